// fft_kernels.cu -- the pseudo-spectral Poisson solve of P:173-177 on sm_100a.
//
//   rho (real, pitched)  --x R2C-->  --y FFT-->  --z FFT, E^_d = -i k_d rho^/|k|^2,
//   3x inverse z-->  --3x inverse y-->  --3x x C2R (+ energy partials)-->  E_d.
//
// Every pass is HBM-bound (about 1.7 flop/B in fp64): each CTA transforms a batch
// of lines (contiguous rows for x; TW adjacent kx columns for y and z, so every
// global access is a contiguous 16*TW-byte run) with a radix-8 Stockham FFT whose
// first stage reads global memory, whose middle stages run in registers with one
// padded shared-memory exchange each, and whose last stage writes global memory;
// twiddles come from a precomputed fp64 table W_n^m, m < n.  The spectral
// multiply and the three inverse z transforms are fused into the z pass, the
// field-energy partial sums into the C2R x pass.
#include <algorithm>
#include <climits>
#include <cstdio>

#include "kernels.h"

namespace pic {

namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 conj2(double2 a) { return make_double2(a.x, -a.y); }


// ---------------------------------------------------------- Stockham FFT --
// Radix-2/4/8 Stockham autosort FFT of nl lines of length len = 2^logn (natural
// order in and out).  Stage s (radix R, Ns = product of the earlier radices):
//   v[r] = in[j + r len/R] * W_{Ns R}^{(j mod Ns) r},  V = DFT_R(v),
//   out[(j / Ns) Ns R + (j mod Ns) + r Ns] = V[r]          (j < len/R).
// Stage 0 (the remainder radix 2 or 4, else 8) reads src(l, e) -- global memory
// or an on-the-fly transform -- and writes shared memory; middle radix-8 stages
// go through registers and one padded shared round trip each; the last stage
// writes dst(l, e, v) (global) or, with DST_SMEM, shared memory in natural order.
// Shared index of element e of line l: l * ls + pidx(e), pidx(e) = e + e/8 (one
// pad per 8 elements keeps the stride-8 writes of radix-8 stages conflict free).
__device__ __forceinline__ int pidx(int e) { return e + (e >> 3); }
__host__ __device__ inline int line_stride(int len) { return len + len / 8 + 1; }
// Line stride of the column passes (TW lines = lanes l of a quarter warp with two
// or more j): stride = 8 / TW (mod 8) puts the 8 lanes of each 128-bit shared
// access phase on 8 distinct 16-byte slots.
__host__ __device__ constexpr int col_stride(int len, int TW) { return len + len / 8 + 8 / TW; }

template <int SIGN>
__device__ __forceinline__ double2 mul_i(double2 a) {   // a * (-i) forward, a * (+i) inverse
    return SIGN < 0 ? make_double2(a.y, -a.x) : make_double2(-a.y, a.x);
}

template <int SIGN>
__device__ __forceinline__ void dft2(double2* v) {
    const double2 a = v[0], b = v[1];
    v[0] = cadd(a, b);
    v[1] = csub(a, b);
}

template <int SIGN>
__device__ __forceinline__ void dft4(double2& a0, double2& a1, double2& a2, double2& a3) {
    const double2 t0 = cadd(a0, a2), t1 = csub(a0, a2);
    const double2 t2 = cadd(a1, a3), t3 = mul_i<SIGN>(csub(a1, a3));
    a0 = cadd(t0, t2);
    a2 = csub(t0, t2);
    a1 = cadd(t1, t3);
    a3 = csub(t1, t3);
}

template <int SIGN>
__device__ __forceinline__ void dft8(double2* v) {
    // X[k] = E[k] + W8^k O[k], X[k+4] = E[k] - W8^k O[k]; E, O = DFT4 of evens, odds
    double2 e0 = v[0], e1 = v[2], e2 = v[4], e3 = v[6];
    double2 o0 = v[1], o1 = v[3], o2 = v[5], o3 = v[7];
    dft4<SIGN>(e0, e1, e2, e3);
    dft4<SIGN>(o0, o1, o2, o3);
    const double h = 0.70710678118654752440084436210485;
    // W8^1 = (1 -+ i)/sqrt2, W8^2 = -+i, W8^3 = (-1 -+ i)/sqrt2
    const double2 w1o1 = SIGN < 0 ? make_double2(h * (o1.x + o1.y), h * (o1.y - o1.x))
                                  : make_double2(h * (o1.x - o1.y), h * (o1.y + o1.x));
    const double2 w2o2 = mul_i<SIGN>(o2);
    const double2 w3o3 = SIGN < 0 ? make_double2(h * (o3.y - o3.x), -h * (o3.x + o3.y))
                                  : make_double2(-h * (o3.x + o3.y), h * (o3.x - o3.y));
    v[0] = cadd(e0, o0); v[4] = csub(e0, o0);
    v[1] = cadd(e1, w1o1); v[5] = csub(e1, w1o1);
    v[2] = cadd(e2, w2o2); v[6] = csub(e2, w2o2);
    v[3] = cadd(e3, w3o3); v[7] = csub(e3, w3o3);
}

template <int SIGN, int R>
__device__ __forceinline__ void dft_r(double2* v) {
    if constexpr (R == 8) dft8<SIGN>(v);
    else if constexpr (R == 4) dft4<SIGN>(v[0], v[1], v[2], v[3]);
    else dft2<SIGN>(v);
}

// tw[m] = W_{N}^m = exp(-2 pi i m / N), m < N; a line of length len uses
// W_len^q = tw[q << tws], tws = log2(N / len).
template <int SIGN>
__device__ __forceinline__ double2 twid(const double2* __restrict__ tw, int q, int tws) {
    const double2 w = __ldg(tw + (q << tws));
    return SIGN < 0 ? w : conj2(w);
}

// v[r] *= W^{jm r << tsh}, r = 1..7, from three table loads (r = 1, 2, 4) and
// four products (w3 = w1 w2, w5 = w1 w4, w6 = w2 w4, w7 = w3 w4).
template <int SIGN>
__device__ __forceinline__ void twiddle8(double2* v, const double2* __restrict__ tw, int jm, int tsh, int tws) {
    const double2 w1 = twid<SIGN>(tw, jm << tsh, tws);
    const double2 w2 = twid<SIGN>(tw, (2 * jm) << tsh, tws);
    const double2 w4 = twid<SIGN>(tw, (4 * jm) << tsh, tws);
    const double2 w3 = cmul(w1, w2);
    v[1] = cmul(v[1], w1);
    v[2] = cmul(v[2], w2);
    v[3] = cmul(v[3], w3);
    v[4] = cmul(v[4], w4);
    v[5] = cmul(v[5], cmul(w1, w4));
    v[6] = cmul(v[6], cmul(w2, w4));
    v[7] = cmul(v[7], cmul(w3, w4));
}

// Work item it -> (line l, butterfly j): ROWS (lines contiguous in memory, the x
// passes) puts consecutive lanes on consecutive j of one line, so every global
// access of a warp is one contiguous run; otherwise (lines = adjacent columns,
// the y and z passes) consecutive lanes take consecutive lines.
template <bool ROWS>
__device__ __forceinline__ void item_lj(int it, int nl, int nj, int lognj, int& l, int& j) {
    if (ROWS) { l = it >> lognj; j = it & (nj - 1); }
    else { l = it % nl; j = it / nl; }
}

// Lines of length 2^LOGN (compile time: every stage's radix, butterfly count and
// twiddle stride are constants).  IPT = middle-stage work items held per thread
// (nl * len <= 8 * IPT * blockDim).
// after0() runs once every thread is past stage 0 (the persistent kernels issue
// the next tile's input copies there: src is no longer read).
struct NoHook {
    __device__ void operator()() const {}
};

template <int SIGN, bool DST_SMEM, int LOGN, int IPT, bool ROWS, class Src, class Dst, class Hook = NoHook>
__device__ __forceinline__ void fft_lines(double2* sm, int nl, int ls, const double2* __restrict__ tw,
                                          int tws, Src src, Dst dst, Hook after0 = Hook()) {
    constexpr int len = 1 << LOGN;
    constexpr int logR0 = LOGN % 3 == 0 ? 3 : LOGN % 3;
    constexpr int nst = (LOGN - logR0) / 3 + 1;
    // ---- stage 0: src -> shared (or dst when it is also the last stage)
    {
        constexpr int R = 1 << logR0, nj = len >> logR0;
        constexpr bool last = nst == 1;
        for (int it = threadIdx.x; it < nl * nj; it += blockDim.x) {
            int l, j;
            item_lj<ROWS>(it, nl, nj, LOGN - logR0, l, j);
            double2 v[R];
#pragma unroll
            for (int r = 0; r < R; ++r) v[r] = src(l, j + r * nj);
            dft_r<SIGN, R>(v);
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int e = j * R + r;        // Ns = 1
                if (last && !DST_SMEM) dst(l, e, v[r]);
                else sm[l * ls + pidx(e)] = v[r];
            }
        }
    }
    __syncthreads();
    after0();
#pragma unroll
    for (int s = 1; s < nst; ++s) {
        const int logNs = logR0 + 3 * (s - 1);
        constexpr int nj = len >> 3;
        const int Ns = 1 << logNs;
        const int tsh = LOGN - logNs - 3;       // W_{Ns 8}^{q} = W_len^{q << tsh}
        const bool last = s == nst - 1;
        if (last && !DST_SMEM) {
            for (int it = threadIdx.x; it < nl * nj; it += blockDim.x) {
                int l, j;
                item_lj<ROWS>(it, nl, nj, LOGN - 3, l, j);
                double2 v[8];
#pragma unroll
                for (int r = 0; r < 8; ++r) v[r] = sm[l * ls + pidx(j + r * nj)];
                const int jm = j & (Ns - 1);
                twiddle8<SIGN>(v, tw, jm, tsh, tws);
                dft8<SIGN>(v);
                const int base = ((j >> logNs) << (logNs + 3)) + jm;
#pragma unroll
                for (int r = 0; r < 8; ++r) dst(l, base + r * Ns, v[r]);
            }
        } else {
            double2 v[IPT][8];
            int lk[IPT], jk[IPT];
#pragma unroll
            for (int k = 0; k < IPT; ++k) {
                const int it = threadIdx.x + k * blockDim.x;
                lk[k] = -1;
                if (it < nl * nj) {
                    int l, j;
                    item_lj<ROWS>(it, nl, nj, LOGN - 3, l, j);
                    lk[k] = l;
                    jk[k] = j;
#pragma unroll
                    for (int r = 0; r < 8; ++r) v[k][r] = sm[l * ls + pidx(j + r * nj)];
                    const int jm = j & (Ns - 1);
                    twiddle8<SIGN>(v[k], tw, jm, tsh, tws);
                    dft8<SIGN>(v[k]);
                }
            }
            __syncthreads();
#pragma unroll
            for (int k = 0; k < IPT; ++k)
                if (lk[k] >= 0) {
                    const int j = jk[k], jm = j & (Ns - 1);
                    const int base = ((j >> logNs) << (logNs + 3)) + jm;
#pragma unroll
                    for (int r = 0; r < 8; ++r) sm[lk[k] * ls + pidx(base + r * Ns)] = v[k][r];
                }
        }
        __syncthreads();
    }
}

__host__ __device__ inline int ilog2(int v) {
    int l = 0;
    while ((1 << l) < v) ++l;
    return l;
}

// Elements per CTA: rows of the x passes, TW columns of the y and z passes.
__host__ __device__ inline int x_rows(int n) { int r = 2048 / (n / 2); return r < 1 ? 1 : r; }
__host__ __device__ inline int xi_rows(int n) { int r = 512 / (n / 2); return r < 1 ? 1 : r; }
__host__ __device__ constexpr int y_tw(int n) { int t = 2048 / n; return t > 8 ? 8 : (t < 1 ? 1 : t); }
__host__ __device__ constexpr int z_tw(int n) { int t = 2048 / n; return t > 8 ? 8 : (t < 1 ? 1 : t); }
// columns per z-pass tile (compile-time knob for A/B: -DPIC_ZMUL_TWN=1024 halves the tile)
#ifndef PIC_ZMUL_TWN
#define PIC_ZMUL_TWN 2048
#endif
#ifndef PIC_ZMUL_MINB
#define PIC_ZMUL_MINB 2
#endif
#ifndef PIC_ZMUL_DIRECT
#define PIC_ZMUL_DIRECT 0
#endif
#ifndef PIC_XINV_DIRECT
#define PIC_XINV_DIRECT 0
#endif
#ifndef PIC_ZMUL_FUSED
#define PIC_ZMUL_FUSED 0
#endif
#ifndef PIC_FFTY_MINB       // resident CTAs per SM the y passes are compiled for
#define PIC_FFTY_MINB 2
#endif
__host__ __device__ constexpr int zmul_tw(int n) { int t = PIC_ZMUL_TWN / n; return t > 8 ? 8 : (t < 1 ? 1 : t); }

// Every pass is a persistent loop over tiles (grid = resident CTAs): the input of
// tile t + gridDim is copied into the shared input buffer with cp.async as soon as
// stage 0 of tile t has consumed it, so the loads of one tile overlap the
// butterflies and stores of the previous one.

// ------------------------------------------------------------ x R2C -------
// Row r of S0 (nzl * n rows): n reals -> n/2 + 1 complex, in place (a tile = R rows).
// z[m] = x[2m] + i x[2m+1] -> Z = FFT_{n/2}(z) -> X[k] = Ze[k] + W_n^k Zo[k],
// Ze = (Z[k] + conj Z[n/2-k])/2, Zo = (Z[k] - conj Z[n/2-k])(-i/2).
template <int LOGN>
__global__ void __launch_bounds__(kThreads, 3) k_fft_x_fwd(Geom g, double* buf,
                                                           const double2* __restrict__ tw) {
    extern __shared__ double2 smx[];
    constexpr int len = 1 << LOGN;
    const int R = x_rows(g.n), ls = line_stride(len);
    double2* in = smx;               // [R][len]
    double2* sm = smx + R * len;     // [R][ls]
    const int64_t nrows = (int64_t)g.nzl * g.n, ntile = (nrows + R - 1) / R;
    auto prefetch = [&](int64_t t) {
        const int64_t row0 = t * R;
        const int rows = (int)min((int64_t)R, nrows - row0);
        for (int i = threadIdx.x; i < rows * len; i += blockDim.x) {
            const int rl = i >> LOGN, e = i & (len - 1);
            cp_async16(in + i, reinterpret_cast<const double2*>(buf + (row0 + rl) * g.rp) + e);
        }
        cp_async_commit();
    };
    int64_t t = blockIdx.x;
    if (t < ntile) prefetch(t);
    for (; t < ntile; t += gridDim.x) {
        const int64_t row0 = t * R;
        const int rows = (int)min((int64_t)R, nrows - row0);
        cp_async_wait0();
        __syncthreads();
        auto src = [&](int l, int e) { return in[l * len + e]; };
        auto dst = [&](int, int, double2) {};
        auto next = [&]() { if (t + gridDim.x < ntile) prefetch(t + gridDim.x); };
        fft_lines<-1, true, LOGN, 1, true>(sm, rows, ls, tw, 1, src, dst, next);
        for (int i = threadIdx.x; i < rows * (len + 1); i += blockDim.x) {
            const int rl = i / (len + 1), k = i - rl * (len + 1);
            const double2 zk = sm[rl * ls + pidx(k & (len - 1))];
            const double2 zc = conj2(sm[rl * ls + pidx((len - k) & (len - 1))]);
            const double2 ze = make_double2(0.5 * (zk.x + zc.x), 0.5 * (zk.y + zc.y));
            const double2 d = csub(zk, zc);
            const double2 zo = make_double2(0.5 * d.y, -0.5 * d.x);
            double2 X;
            if (k == len) X = csub(ze, zo);
            else X = cadd(ze, cmul(__ldg(tw + k), zo));
            reinterpret_cast<double2*>(buf + (row0 + rl) * g.rp)[k] = X;
        }
    }
}

// Element (component d, slab plane zl, row y) of a local spectral layout: row index * px.
__device__ __forceinline__ int64_t spec_row(const Geom& g, const SpecLayout& L, int d, int zl, int y) {
    if (!L.packed) return (((int64_t)d * g.nzl + zl) * g.n + y) * g.px;
    const int q = y >> g.mz, yl = y & (g.nzl - 1);   // nyl = n / P = nzl
    return ((((int64_t)q * L.ncomp + d) * g.nzl + zl) * g.nzl + yl) * g.px;
}

// Row (block q, component d, plane zl, row yl) of a transpose's send side: PACKED
// into this rank's buffer at block q, or REMOTE into rank q's buffer at block rank.
__device__ __forceinline__ double2* xpose_row(const Geom& g, const SpecLayout& L, int q, int d, int zl, int yl) {
    if (L.packed == 2)
        return L.peer[q] + ((((int64_t)g.rank * L.ncomp + d) * g.nzl + zl) * g.nzl + yl) * g.px;
    return L.base + ((((int64_t)q * L.ncomp + d) * g.nzl + zl) * g.nzl + yl) * g.px;
}

// Destination row of element (d, zl, y) of any layout.
__device__ __forceinline__ double2* dst_row(const Geom& g, const SpecLayout& L, int d, int zl, int y) {
    if (!L.packed) return L.base + (((int64_t)d * g.nzl + zl) * g.n + y) * g.px;
    return xpose_row(g, L, y >> g.mz, d, zl, y & (g.nzl - 1));
}

// ------------------------------------------------------------- y pass ------
// Tile (component d, plane zl, kx tile): lines along y of TW consecutive kx columns
// (valid columns kx <= n/2).  A tile's input is all in shared memory before its
// last stage writes, so src and dst may alias.
// EMODE (the inverse pass of the field): the input holds phi^ (component 0) and
// E^_z (component 1), each inverse-z transformed; a phi tile yields two outputs,
// E_x = -i k_x phi (applied to the output, zero on the k_x Nyquist column) and
// E_y = -i k_y phi (applied to the input, zero on the k_y Nyquist row; D#6), an
// E_z tile one.
template <int SIGN, int LOGN, bool EMODE>
__global__ void __launch_bounds__(kThreads, PIC_FFTY_MINB) k_fft_y(Geom g, SpecLayout sl, SpecLayout dl, int ncomp,
                                                       const double2* __restrict__ tw, int64_t tbeg, int64_t tend) {
    extern __shared__ double2 smx[];
    constexpr int n = 1 << LOGN, TW = y_tw(n);
    constexpr int ls = col_stride(n, TW);
    double2* in = smx;               // [n][TW]
    double2* sm = smx + n * TW;      // [TW][ls]
    constexpr int ntiles = (n / 2 + 1 + TW - 1) / TW;
    const int64_t ntile = tend;      // tiles [tbeg, tend) of ncomp * nzl * ntiles (plane-major per component)
    auto prefetch = [&](int64_t t) {
        const int d = (int)(t / ((int64_t)g.nzl * ntiles));
        const int r = (int)(t - (int64_t)d * g.nzl * ntiles);
        const int zl = r / ntiles, kx0 = (r - zl * ntiles) * TW;
        const int ncol = min(TW, n / 2 + 1 - kx0);
        for (int i = threadIdx.x; i < n * TW; i += blockDim.x) {
            const int y = i / TW, l = i % TW;
            if (l < ncol) cp_async16(in + i, sl.base + spec_row(g, sl, d, zl, y) + kx0 + l);
        }
        cp_async_commit();
    };
    const double kf = 6.283185307179586476925286766559 / g.L;
    int64_t t = tbeg + blockIdx.x;
    if (t < ntile) prefetch(t);
    for (; t < ntile; t += gridDim.x) {
        const int d = (int)(t / ((int64_t)g.nzl * ntiles));
        const int r = (int)(t - (int64_t)d * g.nzl * ntiles);
        const int zl = r / ntiles, kx0 = (r - zl * ntiles) * TW;
        const int ncol = min(TW, n / 2 + 1 - kx0);
        cp_async_wait0();
        __syncthreads();
        auto src = [&](int l, int y) { return l < ncol ? in[y * TW + l] : make_double2(0.0, 0.0); };
        auto next = [&]() { if (t + gridDim.x < ntile) prefetch(t + gridDim.x); };
        if (!EMODE) {
            auto dst = [&](int l, int y, double2 v) { if (l < ncol) dst_row(g, dl, d, zl, y)[kx0 + l] = v; };
            fft_lines<SIGN, false, LOGN, 1, false>(sm, TW, ls, tw, 0, src, dst, next);
        } else if (d == 1) {             // E^_z -> E_z
            auto dst = [&](int l, int y, double2 v) { if (l < ncol) dst_row(g, dl, 2, zl, y)[kx0 + l] = v; };
            fft_lines<SIGN, false, LOGN, 1, false>(sm, TW, ls, tw, 0, src, dst, next);
        } else {                         // phi -> (E_x = -i k_x phi, E_y = -i k_y phi)
            auto dst0 = [&](int l, int y, double2 v) {
                if (l < ncol) {
                    const int kx = kx0 + l;       // half spectrum: k_x >= 0; zero on the Nyquist column
                    const double k = kx == n / 2 ? 0.0 : kf * (double)kx;
                    dst_row(g, dl, 0, zl, y)[kx] = make_double2(k * v.y, -k * v.x);
                }
            };
            fft_lines<SIGN, false, LOGN, 1, false>(sm, TW, ls, tw, 0, src, dst0);
            auto srcy = [&](int l, int ky) {
                const double2 v = src(l, ky);
                const double k = ky == n / 2 ? 0.0 : kf * (double)(ky < n / 2 ? ky : ky - n);
                return make_double2(k * v.y, -k * v.x);     // -i k_y phi
            };
            auto dst1 = [&](int l, int y, double2 v) { if (l < ncol) dst_row(g, dl, 1, zl, y)[kx0 + l] = v; };
            fft_lines<SIGN, false, LOGN, 1, false>(sm, TW, ls, tw, 0, srcy, dst1, next);
        }
    }
    if (dl.packed == 2) __threadfence_system();   // peer stores complete before the barrier
}

// --------------------------------------------------- z pass + multiply -----
// Tile (yl, kx tile) of the ky-pencil [z][yl][px] (all n planes, nyl = n / P rows
// of ky, ky = rank nyl + yl).  Forward z FFT of rho^ into shared memory, phi^ =
// rho^ scale / |k|^2 in place (0 at k = 0), then two inverse z FFTs whose first stage
// reads from it: phi^ itself and E^_z = -i k_z phi^ (zero where n_z = -N/2, D#6); the
// x and y components' -i k_d is applied in their own passes.  Stores the two
// components PACKED [q][c][zl][yl][px] (q = z / nzl) for the return transpose (or
// REMOTE).
template <int LOGN>
__global__ void __launch_bounds__(kThreads, PIC_ZMUL_MINB) k_fft_z_mul(Geom g, const double2* __restrict__ pencil,
                                                           SpecLayout out, double scale,
                                                           const double2* __restrict__ tw, int64_t tbeg, int64_t tend) {
    extern __shared__ double2 smx[];
    constexpr int n = 1 << LOGN, TW = zmul_tw(n);
    constexpr int ls = col_stride(n, TW);
    const int nyl = n / g.P;
#if PIC_ZMUL_DIRECT   // stage 0 reads global memory directly: no input buffer (one tile per CTA)
    double2* s1 = smx;               // [TW][ls] forward result
    double2* s2 = s1 + TW * ls;      // [TW][ls] inverse work
    double2* in = nullptr;
#else
    double2* in = smx;               // [n][TW]
    double2* s1 = smx + n * TW;      // [TW][ls] forward result
    double2* s2 = s1 + TW * ls;      // [TW][ls] inverse work
#endif
    constexpr int ntiles = (n / 2 + 1 + TW - 1) / TW;
    const int64_t ntile = tend;      // tiles [tbeg, tend) of nyl * ntiles (ky-row-major)
    const int64_t zstride = (int64_t)nyl * g.px;
    auto prefetch = [&](int64_t t) {
        const int yl = (int)(t / ntiles), kx0 = (int)(t - (int64_t)yl * ntiles) * TW;
        const int ncol = min(TW, n / 2 + 1 - kx0);
        const double2* p = pencil + (int64_t)yl * g.px + kx0;
        for (int i = threadIdx.x; i < n * TW; i += blockDim.x) {
            const int z = i / TW, l = i % TW;
            if (l < ncol) cp_async16(in + i, p + z * zstride + l);
        }
        cp_async_commit();
    };
    const double kf = 6.283185307179586476925286766559 / g.L;
    constexpr int half = n / 2;
    int64_t t = tbeg + blockIdx.x;
#if !PIC_ZMUL_DIRECT
    if (t < ntile) prefetch(t);
#endif
    for (; t < ntile; t += gridDim.x) {
        const int yl = (int)(t / ntiles), kx0 = (int)(t - (int64_t)yl * ntiles) * TW;
        const int ncol = min(TW, n / 2 + 1 - kx0);
        const int ky = g.rank * nyl + yl;
#if PIC_ZMUL_DIRECT
        {
            const double2* pin = pencil + (int64_t)yl * g.px + kx0;
            auto src = [&](int l, int e) { return l < ncol ? pin[e * zstride + l] : make_double2(0.0, 0.0); };
            auto dst = [&](int, int, double2) {};
            fft_lines<-1, true, LOGN, 1, false>(s1, TW, ls, tw, 0, src, dst);
        }
#else
        cp_async_wait0();
        __syncthreads();
        {
            auto src = [&](int l, int e) { return l < ncol ? in[e * TW + l] : make_double2(0.0, 0.0); };
            auto dst = [&](int, int, double2) {};
            auto next = [&]() { if (t + gridDim.x < ntile) prefetch(t + gridDim.x); };
            fft_lines<-1, true, LOGN, 1, false>(s1, TW, ls, tw, 0, src, dst, next);
        }
#endif
        const double kyv = kf * (double)(ky < half ? ky : ky - n);
        // phi^ = rho^ scale / |k|^2 in place (0 at k = 0): one division per mode
        for (int i = threadIdx.x; i < TW * n; i += blockDim.x) {
            const int l = i / n, kz = i % n, kx = kx0 + l;
            const double kxv = kf * (double)(kx < half ? kx : kx - n);
            const double kzv = kf * (double)(kz < half ? kz : kz - n);
            const double k2 = kxv * kxv + kyv * kyv + kzv * kzv;
            const double f = k2 != 0.0 ? scale / k2 : 0.0;
            double2& r = s1[l * ls + pidx(kz)];
            r = make_double2(f * r.x, f * r.y);
        }
        __syncthreads();
#if PIC_ZMUL_FUSED   // both inverse transforms in one fft_lines call: 2 TW lines, two items per thread
        {
            constexpr int ls2 = col_stride(n, 2 * TW);
            auto src = [&](int l, int kz) {
                const int d = l >= TW, lc = l - d * TW;
                double2 e = make_double2(0.0, 0.0);
                if (lc < ncol) {
                    const double2 r = s1[lc * ls + pidx(kz)];
                    if (d == 0) {
                        e = r;                                       // phi^
                    } else if (kz != half) {
                        const double kd = kf * (double)(kz < half ? kz : kz - n);
                        e = make_double2(kd * r.y, -kd * r.x);       // E^_z = -i k_z phi^
                    }
                }
                return e;
            };
            auto dst = [&](int l, int z, double2 v) {
                const int d = l >= TW, lc = l - d * TW;
                if (lc < ncol) {
                    const int q = z >> g.mz, zl = z - (q << g.mz);
                    xpose_row(g, out, q, d, zl, yl)[kx0 + lc] = v;
                }
            };
            fft_lines<+1, false, LOGN, 2, false>(s2, 2 * TW, ls2, tw, 0, src, dst);
            __syncthreads();
        }
#else
        for (int d = 0; d < 2; ++d) {
            auto src = [&](int l, int kz) {
                double2 e = make_double2(0.0, 0.0);
                if (l < ncol) {
                    const double2 r = s1[l * ls + pidx(kz)];
                    if (d == 0) {
                        e = r;                                       // phi^
                    } else if (kz != half) {
                        const double kd = kf * (double)(kz < half ? kz : kz - n);
                        e = make_double2(kd * r.y, -kd * r.x);       // E^_z = -i k_z phi^
                    }
                }
                return e;
            };
            auto dst = [&](int l, int z, double2 v) {
                if (l < ncol) {
                    const int q = z >> g.mz, zl = z - (q << g.mz);
                    xpose_row(g, out, q, d, zl, yl)[kx0 + l] = v;
                }
            };
            fft_lines<+1, false, LOGN, 1, false>(s2, TW, ls, tw, 0, src, dst);
        }
#endif
    }
    if (out.packed == 2) __threadfence_system();
}

// ------------------------------------------------------------ x C2R -------
// A tile = R rows of all three components: n/2 + 1 complex -> n reals each,
// written as node records E4[zl][y][x] = (E_x, E_y, E_z, 0) with 256-bit stores;
// per-CTA partial sums of E_d^2 -> partials[d * gridDim.x + blockIdx.x].
// Z[k] = (X[k] + conj X[n/2-k]) + i (X[k] - conj X[n/2-k]) W_n^{-k} (unnormalised).
__device__ __forceinline__ void st_node(double* p, double a, double b, double c) {
    asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(0.0)
                 : "memory");
}

template <int LOGN>
__global__ void __launch_bounds__(kThreads, 3) k_fft_x_inv(Geom g, const double2* __restrict__ spec,
                                                           double* __restrict__ E4, double* halo,
                                                           const double2* __restrict__ tw,
                                                           double* __restrict__ partials) {
    extern __shared__ double2 smx[];
    __shared__ double red[3][kThreads / 32];
    constexpr int len = 1 << LOGN;
    const int R = xi_rows(g.n), ls = line_stride(len), px = g.px;
#if PIC_XINV_DIRECT   // stage 0 reads the spectra from global memory (L1): no staging buffer
    double2* in = nullptr;
    double2* sm = smx;                   // [3 R][ls]
#else
    double2* in = smx;                   // [3][R][px]
    double2* sm = smx + 3 * R * px;      // [3 R][ls]
#endif
    const int64_t nrows = (int64_t)g.nzl * g.n, ntile = (nrows + R - 1) / R;
    auto prefetch = [&](int64_t t) {
        if (PIC_XINV_DIRECT) return;
        const int64_t row0 = t * R;
        const int per = (int)min((int64_t)R, nrows - row0) * px;
        for (int i = threadIdx.x; i < 3 * per; i += blockDim.x) {
            const int d = i / per, e = i - d * per;
            cp_async16(in + d * R * px + e, spec + ((int64_t)d * nrows + row0) * px + e);
        }
        cp_async_commit();
    };
    double e2[3] = {0.0, 0.0, 0.0};
    int64_t t = blockIdx.x;
    if (t < ntile) prefetch(t);
    for (; t < ntile; t += gridDim.x) {
        const int64_t row0 = t * R;
        const int rows = (int)min((int64_t)R, nrows - row0);
        cp_async_wait0();
        __syncthreads();
        auto src = [&](int l, int k) {          // line l = rl * 3 + d
            const int rl = l / 3, d = l - 3 * rl;
#if PIC_XINV_DIRECT
            const double2* X = spec + ((int64_t)d * nrows + row0 + rl) * px;
            const double2 xk = __ldg(X + k), xc = conj2(__ldg(X + len - k));
#else
            const double2* X = in + (d * R + rl) * px;
            const double2 xk = X[k], xc = conj2(X[len - k]);
#endif
            const double2 ze = cadd(xk, xc);
            const double2 zo = cmul(csub(xk, xc), conj2(__ldg(tw + k)));
            return make_double2(ze.x - zo.y, ze.y + zo.x);
        };
        auto dst = [&](int, int, double2) {};
        auto next = [&]() { if (t + gridDim.x < ntile) prefetch(t + gridDim.x); };
        fft_lines<+1, true, LOGN, 1, true>(sm, 3 * rows, ls, tw, 1, src, dst, next);
        for (int i = threadIdx.x; i < rows * len; i += blockDim.x) {
            const int rl = i >> LOGN, m = i & (len - 1);
            const double2 vx = sm[(3 * rl + 0) * ls + pidx(m)];
            const double2 vy = sm[(3 * rl + 1) * ls + pidx(m)];
            const double2 vz = sm[(3 * rl + 2) * ls + pidx(m)];
            const int64_t nd = 4 * ((row0 + rl) * g.n + 2 * m);
            st_node(E4 + nd, vx.x, vy.x, vz.x);
            st_node(E4 + nd + 4, vx.y, vy.y, vz.y);
            if (halo && row0 + rl < g.n) {      // plane 0 -> the halo plane of the slab below
                st_node(halo + nd, vx.x, vy.x, vz.x);
                st_node(halo + nd + 4, vx.y, vy.y, vz.y);
            }
            e2[0] = fma(vx.x, vx.x, fma(vx.y, vx.y, e2[0]));
            e2[1] = fma(vy.x, vy.x, fma(vy.y, vy.y, e2[1]));
            e2[2] = fma(vz.x, vz.x, fma(vz.y, vz.y, e2[2]));
        }
    }
#pragma unroll
    for (int d = 0; d < 3; ++d) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) e2[d] += __shfl_xor_sync(0xffffffffu, e2[d], o);
        if ((threadIdx.x & 31) == 0) red[d][threadIdx.x >> 5] = e2[d];
    }
    __syncthreads();
    if (threadIdx.x < 3) {
        double s = 0.0;
        for (int w = 0; w < kThreads / 32; ++w) s += red[threadIdx.x][w];
        partials[(int64_t)threadIdx.x * gridDim.x + blockIdx.x] = s;
    }
    if (halo && g.P > 1) __threadfence_system();
}

// compact [nzl][nyl][n] index m <-> node record of E4 [nzl + 1][nyr][n] (pencils skip the
// halo row of every plane)
__device__ __forceinline__ int64_t e4_node(const Geom& g, int64_t m) {
    const int64_t rowc = m >> ilog2(g.n), x = m & (g.n - 1);
    const int64_t zl = rowc / g.nyl, yl = rowc - zl * g.nyl;
    return (zl * g.nyr + yl) * g.n + x;
}

__global__ void k_e4_extract(Geom g, const double* __restrict__ E4, int64_t nn, int d, double* __restrict__ out) {
    const int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (m < nn) out[m] = E4[4 * e4_node(g, m) + d];
}

__global__ void k_e4_pack(Geom g, const double* __restrict__ a, const double* __restrict__ b,
                          const double* __restrict__ c, int64_t nn, double* __restrict__ E4) {
    const int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (m < nn) st_node(E4 + 4 * e4_node(g, m), a[m], b[m], c[m]);
}

// Pencils (pic_api.cu slab_to_pencil_E): the slab field's node records -> the y-group send
// blocks [q][nzs + 1][nyl + 1][n][3] (rows q nyl .. q nyl + nyl, the last one wrapping; 24 B per
// node instead of the 32-B record), and the received blocks -> the pencil's node records.
__global__ void k_e4_pencil_pack(const double* __restrict__ E4s, int n, int nzs, int nyl, int Py,
                                 double* __restrict__ send) {
    const int64_t per = (int64_t)(nzs + 1) * (nyl + 1) * n, tot = per * Py;
    for (int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; m < tot; m += (int64_t)gridDim.x * blockDim.x) {
        const int64_t q = m / per, rem = m - q * per;
        const int x = (int)(rem % n);
        const int64_t pr = rem / n;
        const int r = (int)(pr % (nyl + 1)), p = (int)(pr / (nyl + 1));
        const int y = (int)((q * nyl + r) & (n - 1));
        double ex, ey, ez;
        ldg_node(E4s + 4 * (((int64_t)p * n + y) * n + x), ex, ey, ez);
        double* d = send + 3 * m;
        d[0] = ex;
        d[1] = ey;
        d[2] = ez;
    }
}

__global__ void k_e4_pencil_unpack(const double* __restrict__ recv, int n, int nzs, int nyl, int Py,
                                   double* __restrict__ E4) {
    const int64_t per = (int64_t)(nzs + 1) * (nyl + 1) * n, tot = per * Py;
    for (int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; m < tot; m += (int64_t)gridDim.x * blockDim.x) {
        const int64_t q = m / per, rem = m - q * per;            // from rank q: pencil planes q nzs ..
        const double* s = recv + 3 * m;
        st_node(E4 + 4 * ((int64_t)q * nzs * (nyl + 1) * n + rem), s[0], s[1], s[2]);
    }
}

// Transpose by pulling (peer transport, PIC_XPOSE_PULL=1): rank `rank` copies block `rank` of
// every rank q's send buffer (src_tab[q], mapped over NVLink) to block q of dst -- the
// all-to-all's data movement as one streaming kernel of 16-B loads, four in flight per thread.
__global__ void __launch_bounds__(256) k_xpose_pull(double2* __restrict__ dst, double2* const* __restrict__ src_tab,
                                                    int64_t blk, int rank, int P) {
    const int64_t tot = blk * P, stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 < tot; i0 += 4 * stride) {
        double2 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t i = i0 + u * stride;
            if (i < tot) {
                const int64_t q = i / blk;
                v[u] = __ldcs(src_tab[q] + rank * blk + (i - q * blk));
            }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t i = i0 + u * stride;
            if (i < tot) dst[i] = v[u];
        }
    }
}

// One CTA, fixed summation order (deterministic): energies = (W_x, W).
__global__ void __launch_bounds__(1024) k_energy_reduce(Geom g, const double* __restrict__ partials,
                                                        int nparts, double* __restrict__ energies) {
    __shared__ double red[3][32];
    double s[3] = {0.0, 0.0, 0.0};
    // eight independent loads in flight per thread per round (latency, not bandwidth, bounds one CTA)
    for (int d = 0; d < 3; ++d)
        for (int i0 = threadIdx.x; i0 < nparts; i0 += 8 * blockDim.x) {
            double t[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int i = i0 + u * blockDim.x;
                t[u] = i < nparts ? partials[(int64_t)d * nparts + i] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) s[d] += t[u];
        }
    for (int d = 0; d < 3; ++d) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s[d] += __shfl_xor_sync(0xffffffffu, s[d], o);
        if ((threadIdx.x & 31) == 0) red[d][threadIdx.x >> 5] = s[d];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double t[3];
        for (int d = 0; d < 3; ++d) {
            t[d] = 0.0;
            for (int w = 0; w < (int)(blockDim.x / 32); ++w) t[d] += red[d][w];
        }
        const double h = g.L / (double)g.n;
        const double h3 = (h * h) * h;
        energies[0] = 0.5 * h3 * t[0];
        energies[1] = 0.5 * h3 * (t[0] + t[1] + t[2]);
    }
}

// ---------------------------------------------------- complex 3D FFT ------
// In-place C2C transform of an M^3 complex grid [z][y][x] (M = 2^LOGN <= 1024), one pass
// per axis, unnormalised, sign SIGN (the PIF fine grid: F and F^-1 of P:459-466, DESIGN
// §6f).  A tile of kC2C elements is read whole into shared memory by stage 0 before the
// last stage writes it back, so every pass is in place.  x: kC2C / M contiguous rows;
// y, z: TW = kC2C / M adjacent x columns (each row access one contiguous 16 TW-byte run)
// of one z plane (y pass) or one y row (z pass).  tw = W_M^m, m < M.
constexpr int kC2C = 4096;
__host__ __device__ constexpr int c2c_lines(int M) { return kC2C / M > 8 ? 8 : (kC2C / M < 1 ? 1 : kC2C / M); }

// pmask (nullable): pmask[z] == 0 marks a z plane no one reads (PIF: outside every particle
// tile): the x pass skips its rows, the y pass (mask_outer) the plane.
template <int SIGN, int LOGN>
__global__ void __launch_bounds__(kThreads, 3) k_c2c_rows(double2* __restrict__ g, int64_t nrows,
                                                          const double2* __restrict__ tw,
                                                          const uint32_t* __restrict__ pmask) {
    extern __shared__ double2 smx[];
    constexpr int M = 1 << LOGN, R = c2c_lines(M), ls = M + M / 8 + 1;
    for (int64_t t = blockIdx.x; t * R < nrows; t += gridDim.x) {
        if (pmask && !pmask[(t * R) >> LOGN]) continue;        // R <= M rows: one plane per tile
        double2* base = g + t * R * M;
        const int rows = (int)min((int64_t)R, nrows - t * R);
        auto src = [&](int l, int e) { return base[(int64_t)l * M + e]; };
        auto dst = [&](int l, int e, double2 v) { base[(int64_t)l * M + e] = v; };
        fft_lines<SIGN, false, LOGN, 2, true>(smx, rows, ls, tw, 0, src, dst);
        __syncthreads();
    }
}

// keep > 0: only the lines whose x column (and, with keep_outer, whose outer index) lies in
// [0, keep) or [M - keep, M) are transformed -- the PIF's mode box K_N (keep = N/2): the
// inverse transform's other lines are zero (so skipping them is exact), the forward
// transform's other outputs are never read.
__device__ __forceinline__ bool c2c_in_box(int64_t i, int M, int keep) { return i < keep || i >= M - keep; }

template <int SIGN, int LOGN>
__global__ void __launch_bounds__(kThreads, 3) k_c2c_cols(double2* __restrict__ g, int64_t outer_stride,
                                                          int64_t line_stride_g, const double2* __restrict__ tw,
                                                          int keep, int keep_outer,
                                                          const uint32_t* __restrict__ pmask) {
    extern __shared__ double2 smx[];
    constexpr int M = 1 << LOGN, TW = c2c_lines(M), ls = col_stride(M, TW), nct = M / TW;
    for (int64_t t = blockIdx.x; t < (int64_t)M * nct; t += gridDim.x) {
        const int64_t o = t / nct, ct = t - o * nct;
        if (pmask && !pmask[o]) continue;                       // the y pass: outer = z plane
        if (keep > 0 && ((keep_outer && !c2c_in_box(o, M, keep)) ||
                         !(c2c_in_box(ct * TW, M, keep) || c2c_in_box(ct * TW + TW - 1, M, keep))))
            continue;
        double2* base = g + o * outer_stride + ct * TW;
        auto src = [&](int l, int e) { return base[e * line_stride_g + l]; };
        auto dst = [&](int l, int e, double2 v) { base[e * line_stride_g + l] = v; };
        fft_lines<SIGN, false, LOGN, 2, false>(smx, TW, ls, tw, 0, src, dst);
        __syncthreads();
    }
}

}  // namespace

constexpr int kMaxPartials = 4096;

// Upper bound of the per-CTA energy partials (the x C2R grid), for the workspace.
int energy_partials(const Geom&) { return kMaxPartials; }

// Persistent grid: the resident CTAs of the device (occupancy x SMs), <= ntile.
template <class K>
static unsigned persistent_grid(K kernel, size_t smem, int64_t ntile, int64_t cap = INT32_MAX) {
    int dev = 0, sms = 148, occ = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, kThreads, smem);
    if (occ < 1) occ = 1;
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>(std::min<int64_t>(ntile, cap), (int64_t)occ * sms));
}

// Dispatch on the line length: K = log2(len) of the x passes (len = n/2, n in
// [16, 1024]) and of the y and z passes (len = n).
#define PIC_X_SWITCH(lg, BODY)                                   \
    switch (lg) {                                                \
    case 3: { constexpr int K = 3; BODY; } break;                \
    case 4: { constexpr int K = 4; BODY; } break;                \
    case 5: { constexpr int K = 5; BODY; } break;                \
    case 6: { constexpr int K = 6; BODY; } break;                \
    case 7: { constexpr int K = 7; BODY; } break;                \
    case 8: { constexpr int K = 8; BODY; } break;                \
    case 9: { constexpr int K = 9; BODY; } break;                \
    default: break;                                              \
    }
#define PIC_YZ_SWITCH(lg, BODY)                                  \
    switch (lg) {                                                \
    case 4: { constexpr int K = 4; BODY; } break;                \
    case 5: { constexpr int K = 5; BODY; } break;                \
    case 6: { constexpr int K = 6; BODY; } break;                \
    case 7: { constexpr int K = 7; BODY; } break;                \
    case 8: { constexpr int K = 8; BODY; } break;                \
    case 9: { constexpr int K = 9; BODY; } break;                \
    case 10: { constexpr int K = 10; BODY; } break;              \
    default: break;                                              \
    }

static size_t x_fwd_smem(const Geom& g) {
    const int len = g.n / 2, R = x_rows(g.n);
    return sizeof(double2) * (size_t)R * (len + line_stride(len));
}
static size_t x_inv_smem(const Geom& g) {
    const int len = g.n / 2, R = xi_rows(g.n);
    return sizeof(double2) * 3 * (size_t)R * ((PIC_XINV_DIRECT ? 0 : g.px) + line_stride(len));
}
static int64_t x_tiles(const Geom& g, int R) { return ((int64_t)g.nzl * g.n + R - 1) / R; }

// Grid of the x C2R pass = number of energy partials it writes.
static unsigned x_inv_grid(const Geom& g) {
    const size_t smem = x_inv_smem(g);
    const int64_t nt = x_tiles(g, xi_rows(g.n));
    unsigned grid = 1;
    PIC_X_SWITCH(ilog2(g.n / 2), (grid = persistent_grid(k_fft_x_inv<K>, smem, nt, kMaxPartials)))
    return grid;
}

void launch_fft_x_fwd(const Geom& g, double* S0, const double2* tw, cudaStream_t s) {
    const size_t smem = x_fwd_smem(g);
    const int64_t nt = x_tiles(g, x_rows(g.n));
    PIC_X_SWITCH(ilog2(g.n / 2), (k_fft_x_fwd<K><<<persistent_grid(k_fft_x_fwd<K>, smem, nt), kThreads, smem, s>>>(g, S0, tw)))
}

int fft_plane_tiles(int n) {
    const int TW = y_tw(n);
    return (n / 2 + 1 + TW - 1) / TW;
}
int fft_zrow_tiles(int n) {
    const int TW = zmul_tw(n);
    return (n / 2 + 1 + TW - 1) / TW;
}

void launch_fft_y(const Geom& g, SpecLayout src, SpecLayout dst, int ncomp, int inverse,
                  const double2* tw, cudaStream_t s, int64_t tbeg, int64_t tend) {
    const int TW = y_tw(g.n), ntiles = (g.n / 2 + 1 + TW - 1) / TW;
    const size_t smem = sizeof(double2) * (size_t)TW * (g.n + col_stride(g.n, TW));
    if (tend < 0) tend = (int64_t)ncomp * g.nzl * ntiles;
    const int64_t nt = tend - tbeg;
    if (nt <= 0) return;
    if (inverse)
        PIC_YZ_SWITCH(ilog2(g.n), (k_fft_y<+1, K, false><<<persistent_grid(k_fft_y<+1, K, false>, smem, nt), kThreads, smem, s>>>(g, src, dst, ncomp, tw, tbeg, tend)))
    else
        PIC_YZ_SWITCH(ilog2(g.n), (k_fft_y<-1, K, false><<<persistent_grid(k_fft_y<-1, K, false>, smem, nt), kThreads, smem, s>>>(g, src, dst, ncomp, tw, tbeg, tend)))
}

void launch_fft_y_field(const Geom& g, SpecLayout src, SpecLayout dst, const double2* tw, cudaStream_t s) {
    const int TW = y_tw(g.n), ntiles = (g.n / 2 + 1 + TW - 1) / TW;
    const size_t smem = sizeof(double2) * (size_t)TW * (g.n + col_stride(g.n, TW));
    const int64_t nt = (int64_t)2 * g.nzl * ntiles;
    PIC_YZ_SWITCH(ilog2(g.n), (k_fft_y<+1, K, true><<<persistent_grid(k_fft_y<+1, K, true>, smem, nt), kThreads, smem, s>>>(g, src, dst, 2, tw, 0, nt)))
}

void launch_fft_z_mul(const Geom& g, const double2* pencil, SpecLayout out, double scale,
                      const double2* tw, cudaStream_t s, int64_t tbeg, int64_t tend) {
    const int TW = zmul_tw(g.n), ntiles = (g.n / 2 + 1 + TW - 1) / TW;
    const size_t smem = sizeof(double2) * ((size_t)TW * ((PIC_ZMUL_DIRECT ? 0 : g.n) + col_stride(g.n, TW)) +
                                            (PIC_ZMUL_FUSED ? 2 * (size_t)TW * col_stride(g.n, 2 * TW)
                                                            : (size_t)TW * col_stride(g.n, TW)));
    if (tend < 0) tend = (int64_t)(g.n / g.P) * ntiles;
    const int64_t nt = tend - tbeg;
    if (nt <= 0) return;
    // one tile per CTA: the pass is bound by its four transforms, not its input
    // loads, and measured faster without the persistent loop
    PIC_YZ_SWITCH(ilog2(g.n), (k_fft_z_mul<K><<<(unsigned)nt, kThreads, smem, s>>>(g, pencil, out, scale, tw, tbeg, tend)))
}

void launch_fft_x_inv(const Geom& g, const double2* spec, double* E4, double* halo, const double2* tw,
                      double* partials, cudaStream_t s) {
    const size_t smem = x_inv_smem(g);
    const unsigned grid = x_inv_grid(g);
    PIC_X_SWITCH(ilog2(g.n / 2), (k_fft_x_inv<K><<<grid, kThreads, smem, s>>>(g, spec, E4, halo, tw, partials)))
}

// In-place 3D C2C FFT of an M^3 complex grid, M a power of two in [16, 1024]: x, y, z passes
// forward (sign -1), z, y, x inverse (+1); keep > 0 restricts the y and z passes to the
// lines that meet the box [0, keep) u [M - keep, M) (see c2c_in_box).
cudaError_t launch_fft_c2c_3d(double2* grid, int M, int sign, const double2* tw, cudaStream_t s, int keep,
                              const uint32_t* pmask) {
    const int lg = ilog2(M);
    if ((1 << lg) != M || lg < 4 || lg > 10) return cudaErrorInvalidValue;
    const int64_t M2 = (int64_t)M * M;
    const int R = c2c_lines(M);
    const size_t srow = sizeof(double2) * (size_t)R * (M + M / 8 + 1);
    const size_t scol = sizeof(double2) * (size_t)R * col_stride(M, R);
    const int64_t ntile = M2 * M / ((int64_t)R * M);
    cudaError_t e = cudaSuccess;
#define PIC_C2C_ROWS(SG)                                                                                               \
    (e = cudaFuncSetAttribute(k_c2c_rows<SG, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)srow),              \
     (e == cudaSuccess ? (k_c2c_rows<SG, K><<<persistent_grid(k_c2c_rows<SG, K>, srow, ntile), kThreads, srow, s>>>(   \
          grid, M2, tw, pmask), 0) : 0))
#define PIC_C2C_COLS(SG, OS, LS, KO, PM)                                                                               \
    (e = e == cudaSuccess ? cudaFuncSetAttribute(k_c2c_cols<SG, K>, cudaFuncAttributeMaxDynamicSharedMemorySize,       \
                                                 (int)scol) : e,                                                       \
     (e == cudaSuccess ? (k_c2c_cols<SG, K><<<persistent_grid(k_c2c_cols<SG, K>, scol, ntile), kThreads, scol, s>>>(   \
          grid, OS, LS, tw, keep, KO, PM), 0) : 0))
    if (sign < 0) {
        PIC_YZ_SWITCH(lg, (PIC_C2C_ROWS(-1), PIC_C2C_COLS(-1, M2, (int64_t)M, 0, pmask),
                           PIC_C2C_COLS(-1, (int64_t)M, M2, 1, nullptr)))
    } else {
        PIC_YZ_SWITCH(lg, (PIC_C2C_COLS(+1, (int64_t)M, M2, 1, nullptr), PIC_C2C_COLS(+1, M2, (int64_t)M, 0, pmask),
                           PIC_C2C_ROWS(+1)))
    }
#undef PIC_C2C_ROWS
#undef PIC_C2C_COLS
    return e == cudaSuccess ? cudaGetLastError() : e;
}

void launch_e4_extract(const Geom& g, const double* E4, int d, double* out, cudaStream_t s) {
    const int64_t nn = (int64_t)g.n * g.nyl * g.nzl;
    k_e4_extract<<<(unsigned)((nn + 255) / 256), 256, 0, s>>>(g, E4, nn, d, out);
}

void launch_e4_pack(const Geom& g, const double* const comp[3], double* E4, cudaStream_t s) {
    const int64_t nn = (int64_t)g.n * g.nyl * g.nzl;
    k_e4_pack<<<(unsigned)((nn + 255) / 256), 256, 0, s>>>(g, comp[0], comp[1], comp[2], nn, E4);
}

void launch_e4_pencil_pack(const double* E4s, int n, int nzs, int nyl, int Py, double* send, cudaStream_t s) {
    k_e4_pencil_pack<<<148 * 8, 256, 0, s>>>(E4s, n, nzs, nyl, Py, send);
}

void launch_e4_pencil_unpack(const double* recv, int n, int nzs, int nyl, int Py, double* E4, cudaStream_t s) {
    k_e4_pencil_unpack<<<148 * 8, 256, 0, s>>>(recv, n, nzs, nyl, Py, E4);
}

void launch_xpose_pull(double2* dst, double2* const* src_tab, int64_t blk, int rank, int P, cudaStream_t s) {
    k_xpose_pull<<<148 * 4, 256, 0, s>>>(dst, src_tab, blk, rank, P);
}

void launch_energy_reduce(const Geom& g, const double* partials, double* energies, cudaStream_t s) {
    k_energy_reduce<<<1, 1024, 0, s>>>(g, partials, (int)x_inv_grid(g), energies);
}

// Opt every FFT kernel into > 48 KB of dynamic shared memory (per device: the caller
// runs it once for each device); the first failure is returned.
cudaError_t fft_set_smem_limits() {
    const int big = 200 * 1024;
    cudaError_t e = cudaSuccess;
    auto chk = [&](cudaError_t r) { if (e == cudaSuccess) e = r; };
    for (int lg = 3; lg <= 9; ++lg) {
        PIC_X_SWITCH(lg, (chk(cudaFuncSetAttribute(k_fft_x_fwd<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, big)),
                          chk(cudaFuncSetAttribute(k_fft_x_inv<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, big))))
    }
    for (int lg = 4; lg <= 10; ++lg) {
        PIC_YZ_SWITCH(lg, (chk(cudaFuncSetAttribute(k_fft_y<-1, K, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, big)),
                           chk(cudaFuncSetAttribute(k_fft_y<+1, K, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, big)),
                           chk(cudaFuncSetAttribute(k_fft_y<+1, K, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, big)),
                           chk(cudaFuncSetAttribute(k_fft_z_mul<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, big))))
    }
    return e;
}

}  // namespace pic
