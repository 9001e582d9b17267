// fft_kernels.cu -- the pseudo-spectral Poisson solve of P:173-177 on sm_100a.
//
//   rho (real, pitched)  --x R2C-->  --y FFT-->  --z FFT, E^_d = -i k_d rho^/|k|^2,
//   3x inverse z-->  --3x inverse y-->  --3x x C2R (+ energy partials)-->  E_d.
//
// Every pass is HBM-bound (about 1.7 flop/B in fp64): each CTA stages a batch of
// lines (a contiguous row segment for x, a (line x TW-column) tile for y and z,
// so every global access is a contiguous 16*TW-byte run) in shared memory, runs
// an in-place radix-4 (+ one radix-2) decimation-in-time FFT there with twiddles
// from a precomputed fp64 table, and writes the lines back.  The spectral
// multiply and the three inverse z transforms are fused into the z pass, the
// field-energy partial sums into the C2R x pass.
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

__device__ __forceinline__ unsigned brev(unsigned v, int logn) { return __brev(v) >> (32 - logn); }

// In-place DIT FFT of nl lines of length len = 2^logn in shared memory; line l at
// buf[l*ls ...].  Input in bit-reversed order, output in natural order.
// SIGN = -1: forward e^{-i...}; +1: inverse (unnormalised).  tw[m] = W_M^m with
// M = len << tshift, m < M/2.
template <int SIGN>
__device__ void smem_fft(double2* buf, int nl, int logn, int ls, const double2* __restrict__ tw,
                         int tshift) {
    const int len = 1 << logn;
    int logh = 0;
    if (logn & 1) {  // one radix-2 stage, span 2, twiddle 1
        const int nb = len >> 1;
        for (int t = threadIdx.x; t < nl * nb; t += blockDim.x) {
            const int l = t >> (logn - 1), gi = t & (nb - 1);
            double2* p = buf + l * ls + 2 * gi;
            const double2 a = p[0], b = p[1];
            p[0] = cadd(a, b);
            p[1] = csub(a, b);
        }
        __syncthreads();
        logh = 1;
    }
    // combined radix-2 stages of half-span h and 2h (span 4h), h = 2^logh
    for (; logh < logn; logh += 2) {
        const int h = 1 << logh;
        const int nbl = len >> 2;  // radix-4 butterflies per line
        const int sh1 = logn - logh - 1 + tshift;   // index of W_{2h}^k = k << sh1
        const int sh2 = logn - logh - 2 + tshift;   // index of W_{4h}^k = k << sh2
        for (int t = threadIdx.x; t < nl * nbl; t += blockDim.x) {
            const int l = t >> (logn - 2), r = t & (nbl - 1);
            const int gi = r >> logh, k = r & (h - 1);
            double2* p = buf + l * ls + (gi << (logh + 2)) + k;
            double2 w1 = __ldg(tw + (k << sh1));
            double2 w2 = __ldg(tw + (k << sh2));
            if (SIGN > 0) { w1 = conj2(w1); w2 = conj2(w2); }
            const double2 a0 = p[0], a1 = p[h], a2 = p[2 * h], a3 = p[3 * h];
            const double2 t1 = cmul(a1, w1), t3 = cmul(a3, w1);
            const double2 x0 = cadd(a0, t1), x1 = csub(a0, t1);
            const double2 x2 = cadd(a2, t3), x3 = csub(a2, t3);
            const double2 u2 = cmul(x2, w2);
            double2 u3 = cmul(x3, w2);
            // times -i (forward) or +i (inverse): W_{4h}^h = e^{-/+ i pi/2}
            u3 = SIGN < 0 ? make_double2(u3.y, -u3.x) : make_double2(-u3.y, u3.x);
            p[0] = cadd(x0, u2);
            p[2 * h] = csub(x0, u2);
            p[h] = cadd(x1, u3);
            p[3 * h] = csub(x1, u3);
        }
        __syncthreads();
    }
}

__host__ __device__ inline int ilog2(int v) {
    int l = 0;
    while ((1 << l) < v) ++l;
    return l;
}

// rows per CTA of the x passes (len = n/2 complex per row)
__host__ __device__ inline int x_rows(int n) {
    int r = 4096 / (n / 2);
    return r < 1 ? 1 : r;
}
__host__ __device__ inline int y_tw(int n) { int t = 4096 / n; return t > 8 ? 8 : (t < 1 ? 1 : t); }
__host__ __device__ inline int z_tw(int n) { int t = 2048 / n; return t > 8 ? 8 : (t < 1 ? 1 : t); }

// ------------------------------------------------------------ x R2C -------
// Row r of S0: n reals -> n/2 + 1 complex, in place (the CTA owns its rows).
__global__ void __launch_bounds__(kThreads) k_fft_x_fwd(Geom g, double* buf,
                                                        const double2* __restrict__ tw) {
    extern __shared__ double2 sm[];
    const int len = g.n >> 1, logn = ilog2(len), R = x_rows(g.n), ls = len + 1;
    const int64_t row0 = (int64_t)blockIdx.x * R;
    const int64_t nrows = (int64_t)g.n * g.n;
    const int rows = (int)min((int64_t)R, nrows - row0);
    for (int t = threadIdx.x; t < rows * len; t += blockDim.x) {
        const int rl = t / len, m = t - rl * len;
        const double2* src = reinterpret_cast<const double2*>(buf + (row0 + rl) * g.rp);
        sm[rl * ls + brev(m, logn)] = src[m];
    }
    __syncthreads();
    smem_fft<-1>(sm, rows, logn, ls, tw, 1);
    // X[k] = Ze[k] + W_n^k Zo[k], Ze = (Z[k] + conj Z[len-k])/2, Zo = (Z[k] - conj Z[len-k])(-i/2)
    for (int t = threadIdx.x; t < rows * (len + 1); t += blockDim.x) {
        const int rl = t / (len + 1), k = t - rl * (len + 1);
        const double2 zk = sm[rl * ls + (k & (len - 1))];
        const double2 zc = conj2(sm[rl * ls + ((len - k) & (len - 1))]);
        const double2 ze = make_double2(0.5 * (zk.x + zc.x), 0.5 * (zk.y + zc.y));
        const double2 d = csub(zk, zc);
        const double2 zo = make_double2(0.5 * d.y, -0.5 * d.x);
        double2 X;
        if (k == len) X = csub(ze, zo);
        else X = cadd(ze, cmul(__ldg(tw + k), zo));
        reinterpret_cast<double2*>(buf + (row0 + rl) * g.rp)[k] = X;
    }
}

// ------------------------------------------------------------- y pass ------
// blockIdx.x = z * ntiles + tile, blockIdx.y = component.  Lines along y of TW
// consecutive kx columns (valid columns kx <= n/2).
template <int SIGN>
__global__ void __launch_bounds__(kThreads) k_fft_y(Geom g, double* b0, double* b1, double* b2,
                                                    const double2* __restrict__ tw) {
    extern __shared__ double2 sm[];
    double2* buf = reinterpret_cast<double2*>(blockIdx.y == 0 ? b0 : (blockIdx.y == 1 ? b1 : b2));
    const int n = g.n, logn = ilog2(n), TW = y_tw(n), ls = n + 1;
    const int ntiles = (n / 2 + 1 + TW - 1) / TW;
    const int z = blockIdx.x / ntiles, kx0 = (blockIdx.x - z * ntiles) * TW;
    const int ncol = min(TW, n / 2 + 1 - kx0);
    for (int t = threadIdx.x; t < n * TW; t += blockDim.x) {
        const int y = t / TW, c = t - y * TW;
        if (c < ncol) sm[c * ls + brev(y, logn)] = buf[((int64_t)z * n + y) * g.px + kx0 + c];
    }
    __syncthreads();
    smem_fft<SIGN>(sm, ncol, logn, ls, tw, 0);
    for (int t = threadIdx.x; t < n * TW; t += blockDim.x) {
        const int y = t / TW, c = t - y * TW;
        if (c < ncol) buf[((int64_t)z * n + y) * g.px + kx0 + c] = sm[c * ls + y];
    }
}

// --------------------------------------------------- z pass + multiply -----
// blockIdx.x = ky * ntiles + tile.  Forward z FFT of rho^, then for d = x, y, z:
// E^_d = -i k_d rho^ / |k|^2 * scale (zero at n = 0 and where n_d = -N/2, D#6),
// inverse z FFT, store: E^_x -> S1, E^_y -> S2, E^_z -> S0 (the CTA's own input
// tile, already staged in shared memory).
__global__ void __launch_bounds__(kThreads) k_fft_z_mul(Geom g, double2* rho, double2* e1,
                                                        double2* e2, double scale,
                                                        const double2* __restrict__ tw) {
    extern __shared__ double2 sm[];
    double2* out[3] = {e1, e2, rho};
    const int n = g.n, logn = ilog2(n), TW = z_tw(n), ls = n + 1;
    double2* s1 = sm;
    double2* s2 = sm + TW * ls;
    const int ntiles = (n / 2 + 1 + TW - 1) / TW;
    const int ky = blockIdx.x / ntiles, kx0 = (blockIdx.x - ky * ntiles) * TW;
    const int ncol = min(TW, n / 2 + 1 - kx0);
    const int64_t zstride = (int64_t)n * g.px;
    const int64_t base = (int64_t)ky * g.px + kx0;
    for (int t = threadIdx.x; t < n * TW; t += blockDim.x) {
        const int z = t / TW, c = t - z * TW;
        if (c < ncol) s1[c * ls + brev(z, logn)] = rho[base + z * zstride + c];
    }
    __syncthreads();
    smem_fft<-1>(s1, ncol, logn, ls, tw, 0);
    const double kf = 6.283185307179586476925286766559 / g.L;
    const int half = n / 2;
    const double kyv = kf * (double)(ky < half ? ky : ky - n);
    for (int d = 0; d < 3; ++d) {
        for (int t = threadIdx.x; t < n * TW; t += blockDim.x) {
            const int kz = t / TW, c = t - kz * TW;
            if (c >= ncol) continue;
            const int kx = kx0 + c;
            const double kxv = kf * (double)(kx < half ? kx : kx - n);
            const double kzv = kf * (double)(kz < half ? kz : kz - n);
            const double k2 = kxv * kxv + kyv * kyv + kzv * kzv;
            const int idx = d == 0 ? kx : (d == 1 ? ky : kz);
            const double kd = d == 0 ? kxv : (d == 1 ? kyv : kzv);
            double2 e = make_double2(0.0, 0.0);
            if (k2 != 0.0 && idx != half) {
                const double2 r = s1[c * ls + kz];
                const double f = kd * scale / k2;
                e = make_double2(f * r.y, -f * r.x);   // -i k_d rho^ / |k|^2
            }
            s2[c * ls + brev(kz, logn)] = e;
        }
        __syncthreads();
        smem_fft<+1>(s2, ncol, logn, ls, tw, 0);
        for (int t = threadIdx.x; t < n * TW; t += blockDim.x) {
            const int z = t / TW, c = t - z * TW;
            if (c < ncol) out[d][base + z * zstride + c] = s2[c * ls + z];
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------ x C2R -------
// R rows of all three components per CTA: n/2 + 1 complex -> n reals each,
// written as node records E4[row][x] = (E_x, E_y, E_z, 0) with 256-bit stores;
// per-CTA partial sums of E_d^2 -> partials[d * gridDim.x + blockIdx.x].
__host__ __device__ inline int xi_rows(int n) { int r = 1024 / (n / 2); return r < 1 ? 1 : r; }

__device__ __forceinline__ void st_node(double* p, double a, double b, double c) {
    asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(0.0)
                 : "memory");
}

__global__ void __launch_bounds__(kThreads) k_fft_x_inv(Geom g, const double* b0, const double* b1,
                                                        const double* b2, double* __restrict__ E4,
                                                        const double2* __restrict__ tw,
                                                        double* __restrict__ partials) {
    extern __shared__ double2 sm[];
    __shared__ double red[3][kThreads / 32];
    const int len = g.n >> 1, logn = ilog2(len), R = xi_rows(g.n), ls = len + 1;
    const int64_t row0 = (int64_t)blockIdx.x * R;
    const int rows = (int)min((int64_t)R, (int64_t)g.n * g.n - row0);
    // Z[k] = (X[k] + conj X[len-k]) + i (X[k] - conj X[len-k]) W_n^{-k}, k < len
    for (int t = threadIdx.x; t < 3 * rows * len; t += blockDim.x) {
        const int l = t / len, k = t - l * len;           // line l = d * rows + rl
        const int d = l / rows, rl = l - d * rows;
        const double* buf = d == 0 ? b0 : (d == 1 ? b1 : b2);
        const double2* X = reinterpret_cast<const double2*>(buf + (row0 + rl) * g.rp);
        const double2 xk = X[k], xc = conj2(X[len - k]);
        const double2 ze = cadd(xk, xc);
        const double2 zo = cmul(csub(xk, xc), conj2(__ldg(tw + k)));
        sm[l * ls + brev(k, logn)] = make_double2(ze.x - zo.y, ze.y + zo.x);
    }
    __syncthreads();
    smem_fft<+1>(sm, 3 * rows, logn, ls, tw, 1);
    double e2[3] = {0.0, 0.0, 0.0};
    for (int t = threadIdx.x; t < rows * len; t += blockDim.x) {
        const int rl = t / len, m = t - rl * len;
        const double2 vx = sm[(0 * rows + rl) * ls + m];
        const double2 vy = sm[(1 * rows + rl) * ls + m];
        const double2 vz = sm[(2 * rows + rl) * ls + m];
        double* node = E4 + 4 * ((row0 + rl) * g.n + 2 * m);
        st_node(node, vx.x, vy.x, vz.x);
        st_node(node + 4, vx.y, vy.y, vz.y);
        e2[0] = fma(vx.x, vx.x, fma(vx.y, vx.y, e2[0]));
        e2[1] = fma(vy.x, vy.x, fma(vy.y, vy.y, e2[1]));
        e2[2] = fma(vz.x, vz.x, fma(vz.y, vz.y, e2[2]));
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
}

__global__ void k_e4_extract(const double* __restrict__ E4, int64_t nn, int d, double* __restrict__ out) {
    const int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (m < nn) out[m] = E4[4 * m + d];
}

__global__ void k_e4_pack(const double* __restrict__ a, const double* __restrict__ b,
                          const double* __restrict__ c, int64_t nn, double* __restrict__ E4) {
    const int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (m < nn) st_node(E4 + 4 * m, a[m], b[m], c[m]);
}

// One CTA, fixed summation order (deterministic): energies = (W_x, W).
__global__ void __launch_bounds__(1024) k_energy_reduce(Geom g, const double* __restrict__ partials,
                                                        int nparts, double* __restrict__ energies) {
    __shared__ double red[3][32];
    double s[3] = {0.0, 0.0, 0.0};
    for (int d = 0; d < 3; ++d)
        for (int i = threadIdx.x; i < nparts; i += blockDim.x) s[d] += partials[(int64_t)d * nparts + i];
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

}  // namespace

int energy_partials(const Geom& g) {
    const int64_t nrows = (int64_t)g.n * g.n;
    return (int)((nrows + xi_rows(g.n) - 1) / xi_rows(g.n));
}

void launch_fft_x_fwd(const Geom& g, double* S0, const double2* tw, cudaStream_t s) {
    const int len = g.n / 2, R = x_rows(g.n);
    const size_t smem = sizeof(double2) * (size_t)R * (len + 1);
    const int64_t nrows = (int64_t)g.n * g.n;
    k_fft_x_fwd<<<(unsigned)((nrows + R - 1) / R), kThreads, smem, s>>>(g, S0, tw);
}

void launch_fft_y(const Geom& g, double* const buf[3], int ncomp, int inverse, const double2* tw,
                  cudaStream_t s) {
    const int TW = y_tw(g.n), ntiles = (g.n / 2 + 1 + TW - 1) / TW;
    const size_t smem = sizeof(double2) * (size_t)TW * (g.n + 1);
    dim3 grid(g.n * ntiles, ncomp);
    if (inverse) k_fft_y<+1><<<grid, kThreads, smem, s>>>(g, buf[0], buf[1], buf[2], tw);
    else k_fft_y<-1><<<grid, kThreads, smem, s>>>(g, buf[0], buf[1], buf[2], tw);
}

void launch_fft_z_mul(const Geom& g, double* S0, double* S1, double* S2, double scale,
                      const double2* tw, cudaStream_t s) {
    const int TW = z_tw(g.n), ntiles = (g.n / 2 + 1 + TW - 1) / TW;
    const size_t smem = 2 * sizeof(double2) * (size_t)TW * (g.n + 1);
    k_fft_z_mul<<<g.n * ntiles, kThreads, smem, s>>>(
        g, reinterpret_cast<double2*>(S0), reinterpret_cast<double2*>(S1),
        reinterpret_cast<double2*>(S2), scale, tw);
}

void launch_fft_x_inv(const Geom& g, const double* const spec[3], double* E4, const double2* tw,
                      double* partials, cudaStream_t s) {
    const int len = g.n / 2, R = xi_rows(g.n);
    const size_t smem = 3 * sizeof(double2) * (size_t)R * (len + 1);
    k_fft_x_inv<<<energy_partials(g), kThreads, smem, s>>>(g, spec[0], spec[1], spec[2], E4, tw, partials);
}

void launch_e4_extract(const Geom& g, const double* E4, int d, double* out, cudaStream_t s) {
    const int64_t nn = (int64_t)g.n * g.n * g.n;
    k_e4_extract<<<(unsigned)((nn + 255) / 256), 256, 0, s>>>(E4, nn, d, out);
}

void launch_e4_pack(const Geom& g, const double* const comp[3], double* E4, cudaStream_t s) {
    const int64_t nn = (int64_t)g.n * g.n * g.n;
    k_e4_pack<<<(unsigned)((nn + 255) / 256), 256, 0, s>>>(comp[0], comp[1], comp[2], nn, E4);
}

void launch_energy_reduce(const Geom& g, const double* partials, double* energies, cudaStream_t s) {
    k_energy_reduce<<<1, 1024, 0, s>>>(g, partials, energy_partials(g), energies);
}

// Opt every FFT kernel into > 48 KB of dynamic shared memory once.
void fft_set_smem_limits() {
    const int big = 200 * 1024;
    cudaFuncSetAttribute(k_fft_x_fwd, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    cudaFuncSetAttribute(k_fft_y<-1>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    cudaFuncSetAttribute(k_fft_y<+1>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    cudaFuncSetAttribute(k_fft_z_mul, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    cudaFuncSetAttribute(k_fft_x_inv, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
}

}  // namespace pic
