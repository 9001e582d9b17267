// pif.cu -- Particle-in-Fourier field solve and the type-1 / type-2 NUFFTs on the GPU
// (Appendix A; include/pif.h).
//
// Pipeline (fine grid M = 2N per dimension, complex [lz][ly][lx]):
//   type 1  (D chi F C):  k_spread<W> (one thread per particle, w^3 RED.ADD.F64 on the real
//           parts) -> forward 3D FFT -> k_select (chi, D) or k_pif_modes (chi, D, Poisson,
//           -i k, energy partials).
//   type 2  (C^T F^-1 chi^T D):  k_fill (chi^T D: the selected modes scaled, zero elsewhere)
//           -> inverse 3D FFT -> k_interp<W> (one thread per particle, w^3 loads).
// F is the repo's own radix-8 Stockham FFT (fft_kernels.cu, launch_fft_c2c_3d: one in-place
// pass per axis on the M^3 complex grid), not a library call.
// The PIF solve packs E^_x + i E^_y into one type-2 transform (each is the transform of a
// Hermitian spectrum, hence real) and E^_z into a second.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>

#include "../../include/pif.h"
#include "kernels.h"

namespace {

constexpr int kThreads = 256;
constexpr int kModeBlocks = 1184;      // 148 SMs x 8: the mode kernels' grid (energy partials)
constexpr int kNq = 64;               // Gauss-Legendre nodes for psi^
constexpr int kMaxSteps = 4096;        // pic_pif_step energy history
constexpr int kForward = -1, kInverse = +1;   // F: e^{-i k.x}; F^-1: e^{+i k.x}, unnormalised
thread_local char g_err[256] = "";

__device__ __forceinline__ double psi_es(double z, double beta) {
    // exp(beta (sqrt(1 - z^2) - 1)), |z| <= 1 (D#34); separately rounded ops.
    const double t = __dsub_rn(1.0, __dmul_rn(z, z));
    if (t < 0.0) return 0.0;
    return exp(__dmul_rn(beta, __dsub_rn(sqrt(t), 1.0)));
}

// Fine-grid start index and the W window values of one coordinate (u = x M / L); z = (l - u)
// times 2/W (the oracle divides by W/2: within an ulp, and no fp64 division sequence).
template <int W>
__device__ __forceinline__ int window_1d(double x, double inv_hf, double beta, int M, double* wv) {
    const double u = __dmul_rn(x, inv_hf);
    const double l0d = ceil(__dsub_rn(u, 0.5 * W));
    const int l0 = (int)l0d;
#pragma unroll
    for (int k = 0; k < W; ++k) wv[k] = psi_es(__dmul_rn(__dsub_rn((double)(l0 + k), u), 2.0 / W), beta);
    return l0 < 0 ? l0 + M : l0;
}

__device__ __forceinline__ int wrap_idx(int l, int M) { return l >= M ? l - M : l; }

// C: b_l += f_j psi_z psi_y psi_x, real weights into the real parts.
template <int W>
__global__ void __launch_bounds__(kThreads) k_spread(int64_t np, const double* __restrict__ X,
                                                     const double* __restrict__ f, double* __restrict__ G,
                                                     int M, double inv_hf, double beta) {
    const int64_t j = (int64_t)blockIdx.x * kThreads + threadIdx.x;
    if (j >= np) return;
    double wx[W], wy[W], wz[W];
    const int lx = window_1d<W>(X[j], inv_hf, beta, M, wx);
    const int ly = window_1d<W>(X[np + j], inv_hf, beta, M, wy);
    const int lz = window_1d<W>(X[2 * np + j], inv_hf, beta, M, wz);
    const double fj = f[j];
#pragma unroll 1
    for (int c = 0; c < W; ++c) {
        const int iz = wrap_idx(lz + c, M);
        const double fz = __dmul_rn(fj, wz[c]);
#pragma unroll 1
        for (int b = 0; b < W; ++b) {
            const int iy = wrap_idx(ly + b, M);
            const double fzy = __dmul_rn(fz, wy[b]);
            double* row = G + 2 * (((int64_t)iz * M + iy) * M);
#pragma unroll
            for (int a = 0; a < W; ++a) atomicAdd(row + 2 * wrap_idx(lx + a, M), __dmul_rn(fzy, wx[a]));
        }
    }
}

// C^T: out_j = sum_l g_l psi_z psi_y psi_x.  o_re / o_im nullable, scaled.
template <int W>
__global__ void __launch_bounds__(kThreads) k_interp(int64_t np, const double* __restrict__ X,
                                                     const double2* __restrict__ G, int M, double inv_hf,
                                                     double beta, double* __restrict__ o_re,
                                                     double* __restrict__ o_im, int64_t ostride,
                                                     double scale) {
    const int64_t j = (int64_t)blockIdx.x * kThreads + threadIdx.x;
    if (j >= np) return;
    double wx[W], wy[W], wz[W];
    const int lx = window_1d<W>(X[j], inv_hf, beta, M, wx);
    const int ly = window_1d<W>(X[np + j], inv_hf, beta, M, wy);
    const int lz = window_1d<W>(X[2 * np + j], inv_hf, beta, M, wz);
    double sr = 0.0, si = 0.0;
#pragma unroll 1
    for (int c = 0; c < W; ++c) {
        const int iz = wrap_idx(lz + c, M);
        double yr = 0.0, yi = 0.0;
#pragma unroll 1
        for (int b = 0; b < W; ++b) {
            const int iy = wrap_idx(ly + b, M);
            const double2* row = G + ((int64_t)iz * M + iy) * M;
            double xr = 0.0, xi = 0.0;
#pragma unroll
            for (int a = 0; a < W; ++a) {
                const double2 v = __ldg(row + wrap_idx(lx + a, M));
                xr = fma(v.x, wx[a], xr);
                xi = fma(v.y, wx[a], xi);
            }
            yr = fma(xr, wy[b], yr);
            yi = fma(xi, wy[b], yi);
        }
        sr = fma(yr, wz[c], sr);
        si = fma(yi, wz[c], si);
    }
    if (o_re) o_re[j * ostride] = sr * scale;
    if (o_im) o_im[j * ostride] = si * scale;
}

// 1 / psi^(n), n in [-N/2, N/2): Gauss-Legendre (kNq nodes by Newton on P_kNq) of
// (w/2) int_{-1}^{1} psi(z) cos(pi n w z / M) dz.
__global__ void k_psihat(int N, int M, int W, double beta, double* __restrict__ dinv) {
    __shared__ double zs[kNq], as[kNq];
    const int t = threadIdx.x;
    if (t < kNq) {
        double z = cos(M_PI * (t + 0.75) / (kNq + 0.5));
        double dp = 1.0;
        for (int it = 0; it < 100; ++it) {
            double p0 = 1.0, p1 = z;
            for (int k = 2; k <= kNq; ++k) {
                const double p2 = ((2.0 * k - 1.0) * z * p1 - (k - 1.0) * p0) / k;
                p0 = p1;
                p1 = p2;
            }
            dp = kNq * (z * p1 - p0) / (z * z - 1.0);
            const double dz = p1 / dp;
            z -= dz;
            if (fabs(dz) < 1e-16) break;
        }
        double p0 = 1.0, p1 = z;
        for (int k = 2; k <= kNq; ++k) {
            const double p2 = ((2.0 * k - 1.0) * z * p1 - (k - 1.0) * p0) / k;
            p0 = p1;
            p1 = p2;
        }
        dp = kNq * (z * p1 - p0) / (z * z - 1.0);
        zs[t] = z;
        as[t] = 2.0 / ((1.0 - z * z) * dp * dp);
    }
    __syncthreads();
    for (int i = t; i < N; i += blockDim.x) {
        const double n = (double)(i - N / 2);
        double s = 0.0;
        for (int k = 0; k < kNq; ++k) s += as[k] * psi_es(zs[k], beta) * cos(M_PI * n * zs[k] * W / M);
        dinv[i] = 1.0 / (0.5 * W * s);
    }
}

struct ModeIx {
    int nx, ny, nz;      // n + N/2 in [0, N)
    int64_t fine;        // index of n mod M on the fine grid
};
__device__ __forceinline__ ModeIx mode_ix(int64_t t, int N, int M) {
    ModeIx m;
    m.nx = (int)(t % N);
    const int64_t r = t / N;
    m.ny = (int)(r % N);
    m.nz = (int)(r / N);
    const int h = N / 2;
    const int cx = m.nx - h < 0 ? m.nx - h + M : m.nx - h;
    const int cy = m.ny - h < 0 ? m.ny - h + M : m.ny - h;
    const int cz = m.nz - h < 0 ? m.nz - h + M : m.nz - h;
    m.fine = ((int64_t)cz * M + cy) * M + cx;
    return m;
}

// chi, D (type 1): fhat[t] = B[n mod M] / (psi^_z psi^_y psi^_x).
__global__ void __launch_bounds__(kThreads) k_select(int N, int M, const double2* __restrict__ B,
                                                     const double* __restrict__ dinv, double2* __restrict__ fhat) {
    const int64_t nm = (int64_t)N * N * N;
    for (int64_t t = (int64_t)blockIdx.x * kThreads + threadIdx.x; t < nm; t += (int64_t)gridDim.x * kThreads) {
        const ModeIx m = mode_ix(t, N, M);
        const double d = dinv[m.nz] * dinv[m.ny] * dinv[m.nx];
        const double2 v = B[m.fine];
        fhat[t] = make_double2(v.x * d, v.y * d);
    }
}

// chi, D, Poisson, gradient: rho^ = B D; phi^ = rho^/|k|^2; E^_d = -i k_d phi^,
// zero at k = 0 (D#3) and on the unpaired -N/2 planes (D#36).  A = E^_x + i E^_y, Bz = E^_z;
// block partials of |E^_d|^2 (fixed order).
__global__ void __launch_bounds__(kThreads) k_pif_modes(int N, int M, double kunit, const double2* __restrict__ B,
                                                        const double* __restrict__ dinv, double2* __restrict__ A,
                                                        double2* __restrict__ Bz, double* __restrict__ partials) {
    const int64_t nm = (int64_t)N * N * N;
    double e[3] = {0.0, 0.0, 0.0};
    for (int64_t t = (int64_t)blockIdx.x * kThreads + threadIdx.x; t < nm; t += (int64_t)gridDim.x * kThreads) {
        const ModeIx m = mode_ix(t, N, M);
        const int h = N / 2;
        double2 ex = make_double2(0.0, 0.0), ey = ex, ez = ex;
        const double kx = kunit * (m.nx - h), ky = kunit * (m.ny - h), kz = kunit * (m.nz - h);
        const double k2 = kx * kx + ky * ky + kz * kz;
        if (m.nx > 0 && m.ny > 0 && m.nz > 0 && k2 != 0.0) {
            const double d = dinv[m.nz] * dinv[m.ny] * dinv[m.nx];
            const double2 v = B[m.fine];
            const double pr = v.x * d / k2, pi = v.y * d / k2;
            ex = make_double2(kx * pi, -kx * pr);      // -i k phi
            ey = make_double2(ky * pi, -ky * pr);
            ez = make_double2(kz * pi, -kz * pr);
            e[0] += ex.x * ex.x + ex.y * ex.y;
            e[1] += ey.x * ey.x + ey.y * ey.y;
            e[2] += ez.x * ez.x + ez.y * ez.y;
        }
        A[t] = make_double2(ex.x - ey.y, ex.y + ey.x);
        Bz[t] = ez;
    }
    __shared__ double red[3][kThreads];
    for (int d = 0; d < 3; ++d) red[d][threadIdx.x] = e[d];
    __syncthreads();
    for (int s = kThreads / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s)
            for (int d = 0; d < 3; ++d) red[d][threadIdx.x] += red[d][threadIdx.x + s];
        __syncthreads();
    }
    if (threadIdx.x < 3) partials[blockIdx.x * 3 + threadIdx.x] = red[threadIdx.x][0];
}

// Decomposed PIF (P > 1): the same Poisson step and gradient as k_pif_modes, from the selected
// and deconvolved modes rho^ (k_select, then summed over the ranks), in place: A = rho^ on
// input, E^_x + i E^_y on output; Bz = E^_z; block partials of |E^_d|^2 (fixed order).
__global__ void __launch_bounds__(kThreads) k_pif_field(int N, double kunit, double2* __restrict__ A,
                                                        double2* __restrict__ Bz, double* __restrict__ partials) {
    const int64_t nm = (int64_t)N * N * N;
    double e[3] = {0.0, 0.0, 0.0};
    for (int64_t t = (int64_t)blockIdx.x * kThreads + threadIdx.x; t < nm; t += (int64_t)gridDim.x * kThreads) {
        const int h = N / 2;
        const int nx = (int)(t % N), ny = (int)((t / N) % N), nz = (int)(t / ((int64_t)N * N));
        double2 ex = make_double2(0.0, 0.0), ey = ex, ez = ex;
        const double kx = kunit * (nx - h), ky = kunit * (ny - h), kz = kunit * (nz - h);
        const double k2 = kx * kx + ky * ky + kz * kz;
        if (nx > 0 && ny > 0 && nz > 0 && k2 != 0.0) {
            const double2 v = A[t];
            const double pr = v.x / k2, pi = v.y / k2;
            ex = make_double2(kx * pi, -kx * pr);      // -i k phi
            ey = make_double2(ky * pi, -ky * pr);
            ez = make_double2(kz * pi, -kz * pr);
            e[0] += ex.x * ex.x + ex.y * ex.y;
            e[1] += ey.x * ey.x + ey.y * ey.y;
            e[2] += ez.x * ez.x + ez.y * ez.y;
        }
        A[t] = make_double2(ex.x - ey.y, ex.y + ey.x);
        Bz[t] = ez;
    }
    __shared__ double red[3][kThreads];
    for (int d = 0; d < 3; ++d) red[d][threadIdx.x] = e[d];
    __syncthreads();
    for (int s = kThreads / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s)
            for (int d = 0; d < 3; ++d) red[d][threadIdx.x] += red[d][threadIdx.x + s];
        __syncthreads();
    }
    if (threadIdx.x < 3) partials[blockIdx.x * 3 + threadIdx.x] = red[threadIdx.x][0];
}

__global__ void k_energy(int nblk, const double* __restrict__ partials, double scale, double* __restrict__ out,
                         double* __restrict__ hist) {
    if (threadIdx.x < 3) {
        double s = 0.0;
        for (int b = 0; b < nblk; ++b) s += partials[b * 3 + threadIdx.x];
        out[threadIdx.x] = s * scale;
        if (hist && threadIdx.x == 0) *hist = s * scale;
    }
}

// Leapfrog kick-drift-wrap (D#9; the PIC push): v += qm_dt E; x += v dt; x into [0, L).
__global__ void __launch_bounds__(kThreads) k_pif_push(int64_t np, double* __restrict__ X, double* __restrict__ V,
                                                       const double* __restrict__ E, double qm_dt, double dt,
                                                       double L) {
    const int64_t j = (int64_t)blockIdx.x * kThreads + threadIdx.x;
    if (j >= np) return;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        const int64_t i = d * np + j;
        const double v = __dadd_rn(V[i], __dmul_rn(qm_dt, E[i]));
        double x = __dadd_rn(X[i], __dmul_rn(v, dt));
        if (x >= L) {
            x = __dsub_rn(x, L);
        } else if (x < 0.0) {
            x = __dadd_rn(x, L);
            if (x >= L) x = 0.0;
        }
        V[i] = v;
        X[i] = x;
    }
}

// chi^T D (type 2): G[l] = S[mode(l)] D(mode) where l = n mod M for some n in K_N, else 0.
__global__ void __launch_bounds__(kThreads) k_fill(int N, int M, const double2* __restrict__ S,
                                                   const double* __restrict__ dinv, double2* __restrict__ G) {
    const int64_t nf = (int64_t)M * M * M;
    const int h = N / 2;
    for (int64_t l = (int64_t)blockIdx.x * kThreads + threadIdx.x; l < nf; l += (int64_t)gridDim.x * kThreads) {
        const int lx = (int)(l % M);
        const int64_t r = l / M;
        const int ly = (int)(r % M);
        const int lz = (int)(r / M);
        // n = l for l < N/2, l - M for l >= M - N/2; index n + N/2.
        const int ix = lx < h ? lx + h : (lx >= M - h ? lx - M + h : -1);
        const int iy = ly < h ? ly + h : (ly >= M - h ? ly - M + h : -1);
        const int iz = lz < h ? lz + h : (lz >= M - h ? lz - M + h : -1);
        double2 v = make_double2(0.0, 0.0);
        if ((ix | iy | iz) >= 0) {
            const double d = dinv[iz] * dinv[iy] * dinv[ix];
            const double2 s = S[((int64_t)iz * N + iy) * N + ix];
            v = make_double2(s.x * d, s.y * d);
        }
        G[l] = v;
    }
}


// ------------------------------------------------------------- binned path --
// Particles are counting-sorted into bins of kB^3 fine cells (the fine cell holding u); one
// warp per bin spreads its particles into a private shared-memory tile of T^3 points (the bin
// plus the window's reach, plain read-modify-writes: lanes of one particle touch distinct
// points), then flushes the tile with one RED.ADD.F64 per nonzero point: 216 global atomics
// per particle become ~T^3 / (particles per bin) (6.6 at 8 ppc, W = 6).  Interpolation loads
// the bin's tile of the fine grid into shared memory and sums it thread-per-particle.
constexpr int kB = 8;
template <int W>
struct Tile {
    static constexpr int H = W / 2 + 1;         // tile origin = kB b - H
    static constexpr int T = kB + W + 1;        // tile extent (covers l0 - origin in [0, T - W])
    static constexpr int N3 = T * T * T;
    // Spreading tile strides (doubles).  Padding R = W, P = W^2 (mod 16) makes the 64-bit
    // accesses bank-conflict free but costs occupancy; measured no faster at 512^3 (559 vs
    // 550 ms), so the tile stays dense.
    static constexpr int R = T;
    static constexpr int P = T * T;
    static constexpr int NS = T * P;
};

__device__ __forceinline__ int fine_cell(double x, double inv_hf, int M) {
    const int c = (int)__dmul_rn(x, inv_hf);
    return c < M ? c : M - 1;
}

__global__ void __launch_bounds__(kThreads) k_bin_count(int64_t np, const double* __restrict__ X, int M, int nb,
                                                        double inv_hf, uint32_t* __restrict__ cnt) {
    const int64_t j = (int64_t)blockIdx.x * kThreads + threadIdx.x;
    if (j >= np) return;
    const int bx = fine_cell(X[j], inv_hf, M) / kB, by = fine_cell(X[np + j], inv_hf, M) / kB,
              bz = fine_cell(X[2 * np + j], inv_hf, M) / kB;
    const uint32_t bin = (uint32_t)(((int64_t)bz * nb + by) * nb + bx);
    // warp-aggregated: one atomic per distinct bin among the warp's active lanes
    const unsigned act = __activemask();
    const unsigned grp = __match_any_sync(act, bin);
    if ((threadIdx.x & 31) == __ffs(grp) - 1) atomicAdd(cnt + bin, (uint32_t)__popc(grp));
}

__global__ void __launch_bounds__(kThreads) k_bin_place(int64_t np, const double* __restrict__ X, int M, int nb,
                                                        double inv_hf, uint32_t* __restrict__ cursor,
                                                        uint32_t* __restrict__ perm) {
    const int64_t j = (int64_t)blockIdx.x * kThreads + threadIdx.x;
    if (j >= np) return;
    const int bx = fine_cell(X[j], inv_hf, M) / kB, by = fine_cell(X[np + j], inv_hf, M) / kB,
              bz = fine_cell(X[2 * np + j], inv_hf, M) / kB;
    const uint32_t bin = (uint32_t)(((int64_t)bz * nb + by) * nb + bx);
    // warp-aggregated and order-preserving inside the warp: the lanes of one bin take
    // consecutive slots in lane order, so runs of particles that are contiguous in memory stay
    // contiguous in the bin (coalesced particle reads in the spread / gather)
    const unsigned act = __activemask();
    const unsigned grp = __match_any_sync(act, bin);
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(grp) - 1;
    uint32_t base = 0;
    if (lane == leader) base = atomicAdd(cursor + bin, (uint32_t)__popc(grp));
    base = __shfl_sync(grp, base, leader);
    perm[base + __popc(grp & ((1u << lane) - 1u))] = (uint32_t)j;
}

// Bin z layers holding particles (a bin of kB^3 fine cells at layer bz is nonempty).
__global__ void k_bin_layers(const uint32_t* __restrict__ boffs, int64_t nbins, int nb, uint32_t* __restrict__ lmask) {
    for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nbins; b += (int64_t)gridDim.x * blockDim.x)
        if (boffs[b + 1] > boffs[b]) lmask[b / ((int64_t)nb * nb)] = 1u;
}

// Fine plane z is used if the tile of a nonempty layer reaches it: layer bz's tiles cover planes
// kB bz - H .. kB bz - H + T - 1 (mod M), T = kB + W + 1 (the binned spread / gather tiles).
__global__ void k_plane_mask(const uint32_t* __restrict__ lmask, int nb, int M, int H, int W,
                             uint32_t* __restrict__ pmask) {
    const int z = blockIdx.x * blockDim.x + threadIdx.x;
    if (z >= M) return;
    const int T = kB + W + 1;
    uint32_t used = 0;
    for (int bz = 0; bz < nb && !used; ++bz) {
        const int d = ((z - (kB * bz - H)) % M + M) % M;        // z's offset inside layer bz's reach
        if (d < T) used = lmask[bz];
    }
    pmask[z] = used;
}

// Unwrapped window start and the W values of one coordinate (the same arithmetic as window_1d).
template <int W>
__device__ __forceinline__ int window_raw(double x, double inv_hf, double beta, double* wv, double scale) {
    const double u = __dmul_rn(x, inv_hf);
    const int l0 = (int)ceil(__dsub_rn(u, 0.5 * W));
#pragma unroll
    for (int k = 0; k < W; ++k)
        wv[k] = __dmul_rn(scale, psi_es(__dmul_rn(__dsub_rn((double)(l0 + k), u), 2.0 / W), beta));
    return l0;
}

template <int W>
__global__ void __launch_bounds__(32) k_spread_tiled(const double* __restrict__ X, const double* __restrict__ f,
                                                     int64_t np, const uint32_t* __restrict__ perm,
                                                     const uint32_t* __restrict__ offs, double* __restrict__ G,
                                                     int M, int nb, double inv_hf, double beta) {
    using TL = Tile<W>;
    constexpr int T = TL::T;
    extern __shared__ double smem[];
    double* tile = smem;                        // T planes of P doubles (rows of R)
    double* sw = tile + TL::NS;                 // [32][3][W]: x, y, z weights (q folded into z)
    int* so = (int*)(sw + 32 * 3 * W);          // [32][3] window start - tile origin
    const int bin = blockIdx.x;
    const uint32_t beg = offs[bin], end = offs[bin + 1];
    if (beg == end) return;
    const int lane = threadIdx.x;
    const int bx = bin % nb, by = (bin / nb) % nb, bz = bin / (nb * nb);
    const int ox = kB * bx - TL::H, oy = kB * by - TL::H, oz = kB * bz - TL::H;
    for (int i = lane; i < TL::NS; i += 32) tile[i] = 0.0;
    // this lane's window points pp = lane + 32 i: tile offsets and packed (a, b, c), fixed for
    // every particle (the per-particle part of the index is kb)
    constexpr int NP = (W * W * W + 31) / 32;
    int po[NP], pa[NP];
#pragma unroll
    for (int i = 0; i < NP; ++i) {
        const int pp = min(lane + 32 * i, W * W * W - 1);
        const int a = pp % W, b = (pp / W) % W, c = pp / (W * W);
        po[i] = c * TL::P + b * TL::R + a;
        pa[i] = a | (b << 8) | (c << 16);
    }
    for (uint32_t base = beg; base < end; base += 32) {
        const uint32_t jj = base + lane;
        if (jj < end) {
            const int64_t j = perm[jj];
            double* w = sw + lane * 3 * W;
            // z weights carry q: (q psi_z) psi_y psi_x, the oracle's product order
            so[lane * 3 + 0] = window_raw<W>(X[j], inv_hf, beta, w, 1.0) - ox;
            so[lane * 3 + 1] = window_raw<W>(X[np + j], inv_hf, beta, w + W, 1.0) - oy;
            so[lane * 3 + 2] = window_raw<W>(X[2 * np + j], inv_hf, beta, w + 2 * W, f[j]) - oz;
        }
        __syncwarp();
        const int cnt = (int)min(32u, end - base);
        for (int k = 0; k < cnt; ++k) {
            const int kb = so[k * 3 + 2] * TL::P + so[k * 3 + 1] * TL::R + so[k * 3];
            const double* w = sw + k * 3 * W;
            // all loads (window values, then the tile points) before any store, so the NP
            // independent read-modify-writes overlap (the compiler cannot prove that a tile
            // store does not alias the staged window values)
            double val[NP], old[NP];
#pragma unroll
            for (int i = 0; i < NP; ++i) {
                const int a = pa[i] & 0xff, b = (pa[i] >> 8) & 0xff, c = pa[i] >> 16;
                val[i] = __dmul_rn(__dmul_rn(w[2 * W + c], w[W + b]), w[a]);
            }
#pragma unroll
            for (int i = 0; i < NP; ++i) old[i] = tile[kb + po[i]];
#pragma unroll
            for (int i = 0; i < NP; ++i)
                if (i < NP - 1 || lane + 32 * i < W * W * W) tile[kb + po[i]] = __dadd_rn(old[i], val[i]);
            __syncwarp();
        }
    }
    __syncwarp();
    for (int i = lane; i < TL::N3; i += 32) {
        const int tx = i % T, ty = (i / T) % T, tz = i / (T * T);
        const double v = tile[tz * TL::P + ty * TL::R + tx];
        if (v != 0.0) {
            int gx = ox + tx, gy = oy + ty, gz = oz + tz;
            gx = gx < 0 ? gx + M : (gx >= M ? gx - M : gx);
            gy = gy < 0 ? gy + M : (gy >= M ? gy - M : gy);
            gz = gz < 0 ? gz + M : (gz >= M ? gz - M : gz);
            atomicAdd(G + 2 * (((int64_t)gz * M + gy) * M + gx), v);   // real part of the interleaved complex
        }
    }
}

template <int W>
__global__ void __launch_bounds__(128) k_interp_tiled(const double* __restrict__ X, int64_t np,
                                                      const uint32_t* __restrict__ perm,
                                                      const uint32_t* __restrict__ offs,
                                                      const double2* __restrict__ G, int M, int nb, double inv_hf,
                                                      double beta, double* __restrict__ o_re,
                                                      double* __restrict__ o_im, int64_t ostride, double scale) {
    using TL = Tile<W>;
    constexpr int T = TL::T;
    extern __shared__ double2 gt[];             // T^3 complex
    const int bin = blockIdx.x;
    const uint32_t beg = offs[bin], end = offs[bin + 1];
    if (beg == end) return;
    const int bx = bin % nb, by = (bin / nb) % nb, bz = bin / (nb * nb);
    const int ox = kB * bx - TL::H, oy = kB * by - TL::H, oz = kB * bz - TL::H;
    for (int i = threadIdx.x; i < TL::N3; i += blockDim.x) {
        int gx = ox + i % T, gy = oy + (i / T) % T, gz = oz + i / (T * T);
        gx = gx < 0 ? gx + M : (gx >= M ? gx - M : gx);
        gy = gy < 0 ? gy + M : (gy >= M ? gy - M : gy);
        gz = gz < 0 ? gz + M : (gz >= M ? gz - M : gz);
        gt[i] = __ldg(G + ((int64_t)gz * M + gy) * M + gx);
    }
    __syncthreads();
    for (uint32_t jj = beg + threadIdx.x; jj < end; jj += blockDim.x) {
        const int64_t j = perm[jj];
        double wx[W], wy[W], wz[W];
        const int kx = window_raw<W>(X[j], inv_hf, beta, wx, 1.0) - ox;
        const int ky = window_raw<W>(X[np + j], inv_hf, beta, wy, 1.0) - oy;
        const int kz = window_raw<W>(X[2 * np + j], inv_hf, beta, wz, 1.0) - oz;
        double sr = 0.0, si = 0.0;
#pragma unroll 1
        for (int c = 0; c < W; ++c) {
            double yr = 0.0, yi = 0.0;
#pragma unroll
            for (int b = 0; b < W; ++b) {
                const double2* row = gt + ((kz + c) * T + (ky + b)) * T + kx;
                double xr = 0.0, xi = 0.0;
#pragma unroll
                for (int a = 0; a < W; ++a) {
                    const double2 v = row[a];
                    xr = fma(v.x, wx[a], xr);
                    xi = fma(v.y, wx[a], xi);
                }
                yr = fma(xr, wy[b], yr);
                yi = fma(xi, wy[b], yi);
            }
            sr = fma(yr, wz[c], sr);
            si = fma(yi, wz[c], si);
        }
        if (o_re) o_re[j * ostride] = sr * scale;
        if (o_im) o_im[j * ostride] = si * scale;
    }
}


// PIF gather of all three components in one pass (binned path): tile of G1 = E_x + i E_y
// (complex) and of the real part of G2 = E_z; the window is computed once per particle.
template <int W>
__global__ void __launch_bounds__(256) k_interp3_tiled(const double* __restrict__ X, int64_t np,
                                                       const uint32_t* __restrict__ perm,
                                                       const uint32_t* __restrict__ offs,
                                                       const double2* __restrict__ G1,
                                                       const double2* __restrict__ G2, int M, int nb,
                                                       double inv_hf, double beta, double* __restrict__ E,
                                                       double scale) {
    using TL = Tile<W>;
    constexpr int T = TL::T;
    extern __shared__ double2 g1[];             // T^3 complex, then T^3 real
    double* g2 = (double*)(g1 + TL::N3);
    const int bin = blockIdx.x;
    const uint32_t beg = offs[bin], end = offs[bin + 1];
    if (beg == end) return;
    const int bx = bin % nb, by = (bin / nb) % nb, bz = bin / (nb * nb);
    const int ox = kB * bx - TL::H, oy = kB * by - TL::H, oz = kB * bz - TL::H;
    for (int i = threadIdx.x; i < TL::N3; i += blockDim.x) {
        int gx = ox + i % T, gy = oy + (i / T) % T, gz = oz + i / (T * T);
        gx = gx < 0 ? gx + M : (gx >= M ? gx - M : gx);
        gy = gy < 0 ? gy + M : (gy >= M ? gy - M : gy);
        gz = gz < 0 ? gz + M : (gz >= M ? gz - M : gz);
        const int64_t gi = ((int64_t)gz * M + gy) * M + gx;
        g1[i] = __ldg(G1 + gi);
        g2[i] = __ldg((const double*)(G2 + gi));
    }
    __syncthreads();
    for (uint32_t jj = beg + threadIdx.x; jj < end; jj += blockDim.x) {
        const int64_t j = perm[jj];
        double wx[W], wy[W], wz[W];
        const int kx = window_raw<W>(X[j], inv_hf, beta, wx, 1.0) - ox;
        const int ky = window_raw<W>(X[np + j], inv_hf, beta, wy, 1.0) - oy;
        const int kz = window_raw<W>(X[2 * np + j], inv_hf, beta, wz, 1.0) - oz;
        double sr = 0.0, si = 0.0, sz = 0.0;
#pragma unroll 1
        for (int c = 0; c < W; ++c) {
            double yr = 0.0, yi = 0.0, yz = 0.0;
#pragma unroll
            for (int b = 0; b < W; ++b) {
                const int r = ((kz + c) * T + (ky + b)) * T + kx;
                double xr = 0.0, xi = 0.0, xz = 0.0;
#pragma unroll
                for (int a = 0; a < W; ++a) {
                    const double2 v = g1[r + a];
                    xr = fma(v.x, wx[a], xr);
                    xi = fma(v.y, wx[a], xi);
                    xz = fma(g2[r + a], wx[a], xz);
                }
                yr = fma(xr, wy[b], yr);
                yi = fma(xi, wy[b], yi);
                yz = fma(xz, wy[b], yz);
            }
            sr = fma(yr, wz[c], sr);
            si = fma(yi, wz[c], si);
            sz = fma(yz, wz[c], sz);
        }
        E[j] = sr * scale;
        E[np + j] = si * scale;
        E[2 * np + j] = sz * scale;
    }
}

inline size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }

}  // namespace

struct pic_pif {
    int n, M, w;
    double L, eps, beta, inv_hf;
    cudaStream_t stream;
    double2* tw;         // M twiddles W_M^m = exp(-2 pi i m / M) of the fine-grid FFT
    ncclComm_t comm;     // decomposed PIF (pic_pif_attach_nccl): the modes are summed over the ranks
    int nranks;
    double2* G;          // fine grid M^3
    double2* G2;         // second fine grid (binned PIF solve: E_z), or null
    double2* A;          // N^3 spectrum (E^_x + i E^_y)
    double2* Bz;         // N^3 spectrum (E^_z)
    double* dinv;        // N: 1 / psi^
    double* partials;    // kModeBlocks x 3
    double* energy;      // 3
    double* hist;        // kMaxSteps: W_x per step of pic_pif_step
    int hist_slot;       // -1: no history write
    int64_t np_max;      // binned path capacity (0: atomic path only)
    int nb;              // bins per dimension (M / kB)
    bool binned;         // binned spread / interp in use
    bool split_interp;   // PIC_PIF_SPLIT_INTERP=1: two gather passes (E_x + i E_y, then E_z)
    uint32_t* bcnt;      // nb^3 + 1 counts -> offsets
    uint32_t* boffs;     // nb^3 + 1 offsets (exclusive scan)
    uint32_t* bcur;      // nb^3 cursors
    uint32_t* perm;      // np_max particle indices in bin order
    void* scan_tmp;
    size_t scan_bytes;
    uint32_t* pmask;     // [M] fine-grid z planes reached by the binned particles' tiles
    uint32_t* lmask;     // [nb] bin z layers holding particles
    bool poisoned;
    bool timing;
    cudaEvent_t ev[512];
    int nev;
    double ms[PIC_PIF_NSTAGES];
    int64_t launches[PIC_PIF_NSTAGES];
    int ev_stage[256];
    char err[256];
};

namespace {

int width_of(double eps) { return (int)std::ceil(std::log10(1.0 / eps)) + 2; }

// The fine grid M = 2n must be a power of two the FFT passes handle (16 .. 1024).
bool valid(int32_t n, double L, double eps) {
    return n >= 8 && n <= 512 && (n & (n - 1)) == 0 && L > 0 && eps >= 1e-14 && eps < 1.0;
}

struct Layout {
    size_t G, A, Bz, dinv, partials, energy, hist, tw, bcnt, boffs, bcur, perm, scan, pmask, G2, total;
};
bool binnable(int n, int w) { return (2 * n) % kB == 0 && w <= 8; }
// the bins' exclusive scan is the PIC path's own (particle_kernels.cu launch_scan)
size_t scan_tmp_bytes(int64_t nbins) { return pic::scan_scratch_bytes(nbins); }
Layout layout(int n, int64_t np_max, int w) {
    const size_t M = 2 * (size_t)n;
    Layout o;
    size_t off = 0;
    o.G = off;        off += align256(M * M * M * sizeof(double2));
    o.A = off;        off += align256((size_t)n * n * n * sizeof(double2));
    o.Bz = off;       off += align256((size_t)n * n * n * sizeof(double2));
    o.dinv = off;     off += align256((size_t)n * sizeof(double));
    o.partials = off; off += align256((size_t)kModeBlocks * 3 * sizeof(double));
    o.energy = off;   off += align256(3 * sizeof(double));
    o.hist = off;     off += align256(kMaxSteps * sizeof(double));
    o.tw = off;       off += align256(M * sizeof(double2));
    const int64_t nbins = (np_max > 0 && binnable(n, w)) ? (int64_t)(M / kB) * (M / kB) * (M / kB) : 0;
    o.bcnt = off;     off += nbins ? align256((nbins + 1) * 4) : 0;
    o.boffs = off;    off += nbins ? align256((nbins + 1) * 4) : 0;
    o.bcur = off;     off += nbins ? align256(nbins * 4) : 0;
    o.perm = off;     off += nbins ? align256((size_t)np_max * 4) : 0;
    o.scan = off;     off += nbins ? align256(scan_tmp_bytes(nbins)) : 0;
    o.pmask = off;    off += nbins ? align256((M + (M / kB)) * sizeof(uint32_t)) : 0;
    o.G2 = off;       off += nbins ? align256(M * M * M * sizeof(double2)) : 0;
    o.total = off;
    return o;
}

#define PIF_CUDA(p, call)                                                                      \
    do {                                                                                       \
        cudaError_t e_ = (call);                                                               \
        if (e_ != cudaSuccess) {                                                               \
            snprintf((p)->err, sizeof((p)->err), "%s: %s", #call, cudaGetErrorString(e_));     \
            (p)->poisoned = true;                                                              \
            return PIC_ECUDA;                                                                  \
        }                                                                                      \
    } while (0)
#define PIF_LAUNCHED(p)                                                                        \
    do {                                                                                       \
        cudaError_t e_ = cudaGetLastError();                                                   \
        if (e_ != cudaSuccess) {                                                               \
            snprintf((p)->err, sizeof((p)->err), "launch: %s", cudaGetErrorString(e_));        \
            (p)->poisoned = true;                                                              \
            return PIC_ECUDA;                                                                  \
        }                                                                                      \
    } while (0)

struct Stage {
    pic_pif* p;
    int s;
    Stage(pic_pif* p_, int s_) : p(p_), s(s_) {
        p->launches[s] += 1;
        if (p->timing && p->nev + 2 <= (int)(sizeof(p->ev) / sizeof(p->ev[0]))) {
            p->ev_stage[p->nev / 2] = s;
            cudaEventRecord(p->ev[p->nev], p->stream);
        }
    }
    ~Stage() {
        if (p->timing && p->nev + 2 <= (int)(sizeof(p->ev) / sizeof(p->ev[0]))) {
            cudaEventRecord(p->ev[p->nev + 1], p->stream);
            p->nev += 2;
        }
    }
};

#define PIC_TRY_PIF(expr)                   \
    do {                                    \
        pic_status s_ = (expr);             \
        if (s_ != PIC_OK) return s_;        \
    } while (0)

pic_status flush_timing(pic_pif* p) {
    if (!p->timing) return PIC_OK;
    PIF_CUDA(p, cudaStreamSynchronize(p->stream));
    for (int i = 0; i < p->nev; i += 2) {
        float t = 0.f;
        PIF_CUDA(p, cudaEventElapsedTime(&t, p->ev[i], p->ev[i + 1]));
        p->ms[p->ev_stage[i / 2]] += t;
    }
    p->nev = 0;
    return PIC_OK;
}

unsigned particle_grid(int64_t np) { return (unsigned)((np + kThreads - 1) / kThreads); }
unsigned stream_grid(int64_t n) {
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + kThreads - 1) / kThreads, 148 * 16));
}

template <int W>
void spread_w(pic_pif* p, int64_t np, const double* X, const double* f) {
    k_spread<W><<<particle_grid(np), kThreads, 0, p->stream>>>(np, X, f, (double*)p->G, p->M, p->inv_hf, p->beta);
}
template <int W>
void interp_w(pic_pif* p, int64_t np, const double* X, double* ore, double* oim, int64_t os, double sc) {
    k_interp<W><<<particle_grid(np), kThreads, 0, p->stream>>>(np, X, p->G, p->M, p->inv_hf, p->beta, ore, oim,
                                                                 os, sc);
}

#define PIF_W_SWITCH(w, F, ...)                      \
    switch (w) {                                     \
        case 3: F<3>(__VA_ARGS__); break;            \
        case 4: F<4>(__VA_ARGS__); break;            \
        case 5: F<5>(__VA_ARGS__); break;            \
        case 6: F<6>(__VA_ARGS__); break;            \
        case 7: F<7>(__VA_ARGS__); break;            \
        case 8: F<8>(__VA_ARGS__); break;            \
        case 9: F<9>(__VA_ARGS__); break;            \
        case 10: F<10>(__VA_ARGS__); break;          \
        case 11: F<11>(__VA_ARGS__); break;          \
        case 12: F<12>(__VA_ARGS__); break;          \
        case 13: F<13>(__VA_ARGS__); break;          \
        case 14: F<14>(__VA_ARGS__); break;          \
        case 15: F<15>(__VA_ARGS__); break;          \
        default: F<16>(__VA_ARGS__); break;          \
    }

template <int W>
void spread_tiled_w(pic_pif* p, int64_t np, const double* X, const double* f) {
    const size_t sm = (Tile<W>::NS + 32 * 3 * W) * sizeof(double) + 32 * 3 * sizeof(int);
    cudaFuncSetAttribute(k_spread_tiled<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    const int nbins = p->nb * p->nb * p->nb;
    k_spread_tiled<W><<<nbins, 32, sm, p->stream>>>(X, f, np, p->perm, p->boffs, (double*)p->G, p->M, p->nb,
                                                    p->inv_hf, p->beta);
}
template <int W>
void interp_tiled_w(pic_pif* p, int64_t np, const double* X, double* ore, double* oim, int64_t os, double sc) {
    const size_t sm = Tile<W>::N3 * sizeof(double2);
    cudaFuncSetAttribute(k_interp_tiled<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    const int nbins = p->nb * p->nb * p->nb;
    k_interp_tiled<W><<<nbins, 128, sm, p->stream>>>(X, np, p->perm, p->boffs, p->G, p->M, p->nb, p->inv_hf,
                                                     p->beta, ore, oim, os, sc);
}
template <int W>
void interp3_tiled_w(pic_pif* p, int64_t np, const double* X, double* E, double sc) {
    const size_t sm = Tile<W>::N3 * (sizeof(double2) + sizeof(double));
    cudaFuncSetAttribute(k_interp3_tiled<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    const int nbins = p->nb * p->nb * p->nb;
    k_interp3_tiled<W><<<nbins, 256, sm, p->stream>>>(X, np, p->perm, p->boffs, p->G, p->G2, p->M, p->nb,
                                                      p->inv_hf, p->beta, E, sc);
}
#define PIF_W_SWITCH_SMALL(w, F, ...)                \
    switch (w) {                                     \
        case 3: F<3>(__VA_ARGS__); break;            \
        case 4: F<4>(__VA_ARGS__); break;            \
        case 5: F<5>(__VA_ARGS__); break;            \
        case 6: F<6>(__VA_ARGS__); break;            \
        case 7: F<7>(__VA_ARGS__); break;            \
        default: F<8>(__VA_ARGS__); break;           \
    }

// Counting sort of the particles into bins (perm, boffs) for the binned kernels.
pic_status bin(pic_pif* p, int64_t np, const double* X) {
    p->binned = false;
    if (!p->perm || np <= 0 || np > p->np_max) return PIC_OK;
    Stage t(p, PIC_PIF_BIN);
    const int64_t nbins = (int64_t)p->nb * p->nb * p->nb;
    PIF_CUDA(p, cudaMemsetAsync(p->bcnt, 0, (nbins + 1) * sizeof(uint32_t), p->stream));
    k_bin_count<<<particle_grid(np), kThreads, 0, p->stream>>>(np, X, p->M, p->nb, p->inv_hf, p->bcnt);
    PIF_LAUNCHED(p);
    pic::launch_scan(p->bcnt, p->boffs, nbins, (uint32_t*)p->scan_tmp, p->stream);
    PIF_LAUNCHED(p);
    // the fine-grid planes the particles' bin tiles reach (decomposed PIF: a rank's particles
    // occupy a few planes, the x and y passes skip the others)
    PIF_CUDA(p, cudaMemsetAsync(p->lmask, 0, p->nb * sizeof(uint32_t), p->stream));
    k_bin_layers<<<(unsigned)std::max<int64_t>(1, std::min<int64_t>((nbins + kThreads - 1) / kThreads, 148 * 8)),
                   kThreads, 0, p->stream>>>(p->boffs, nbins, p->nb, p->lmask);
    k_plane_mask<<<(p->M + kThreads - 1) / kThreads, kThreads, 0, p->stream>>>(p->lmask, p->nb, p->M,
                                                                              p->w / 2 + 1, p->w, p->pmask);
    PIF_LAUNCHED(p);
    PIF_CUDA(p, cudaMemcpyAsync(p->bcur, p->boffs, nbins * sizeof(uint32_t), cudaMemcpyDeviceToDevice, p->stream));
    k_bin_place<<<particle_grid(np), kThreads, 0, p->stream>>>(np, X, p->M, p->nb, p->inv_hf, p->bcur, p->perm);
    PIF_LAUNCHED(p);
    p->binned = true;
    return PIC_OK;
}

pic_status spread(pic_pif* p, int64_t np, const double* X, const double* f) {
    Stage t(p, PIC_PIF_SPREAD);
    const size_t M = p->M;
    PIF_CUDA(p, cudaMemsetAsync(p->G, 0, M * M * M * sizeof(double2), p->stream));
    if (np > 0) {
        if (p->binned) {
            PIF_W_SWITCH_SMALL(p->w, spread_tiled_w, p, np, X, f);
        } else {
            PIF_W_SWITCH(p->w, spread_w, p, np, X, f);
        }
    }
    PIF_LAUNCHED(p);
    return PIC_OK;
}

pic_status fft(pic_pif* p, int dir, double2* grid = nullptr) {
    Stage t(p, PIC_PIF_FFT);
    double2* g = grid ? grid : p->G;
    // only the lines that meet the mode box K_N: the inverse transform's input is zero
    // outside it (k_fill), the forward transform's output is read only inside it
    PIF_CUDA(p, pic::launch_fft_c2c_3d(g, p->M, dir, p->tw, p->stream, p->n / 2, p->binned ? p->pmask : nullptr));
    return PIC_OK;
}

pic_status fill(pic_pif* p, const double2* S, double2* grid = nullptr) {
    Stage t(p, PIC_PIF_FILL);
    const int64_t nf = (int64_t)p->M * p->M * p->M;
    k_fill<<<stream_grid(nf), kThreads, 0, p->stream>>>(p->n, p->M, S, p->dinv, grid ? grid : p->G);
    PIF_LAUNCHED(p);
    return PIC_OK;
}

pic_status interp(pic_pif* p, int64_t np, const double* X, double* ore, double* oim, int64_t os, double sc) {
    Stage t(p, PIC_PIF_INTERP);
    if (np > 0) {
        if (p->binned) {
            PIF_W_SWITCH_SMALL(p->w, interp_tiled_w, p, np, X, ore, oim, os, sc);
        } else {
            PIF_W_SWITCH(p->w, interp_w, p, np, X, ore, oim, os, sc);
        }
    }
    PIF_LAUNCHED(p);
    return PIC_OK;
}

#define PIF_CHECK(p)                             \
    do {                                         \
        if (!(p)) return PIC_EINVAL;             \
        if ((p)->poisoned) return PIC_EPOISONED; \
    } while (0)

}  // namespace

extern "C" {

pic_status pic_pif_workspace_bytes(int32_t n, double length, double eps, int64_t np_max, size_t* bytes) {
    if (!bytes || !valid(n, length, eps) || np_max < 0 || np_max > (int64_t)UINT32_MAX) {
        snprintf(g_err, sizeof(g_err), "pic_pif_workspace_bytes: invalid n / length / eps");
        return PIC_EINVAL;
    }
    *bytes = layout(n, np_max, width_of(eps)).total;
    return PIC_OK;
}

pic_status pic_pif_create(int32_t n, double length, double eps, int64_t np_max, void* workspace, size_t bytes,
                          void* stream, pic_pif** out) {
    if (!out || !workspace || !valid(n, length, eps) || np_max < 0 || np_max > (int64_t)UINT32_MAX) {
        snprintf(g_err, sizeof(g_err), "pic_pif_create: invalid argument");
        return PIC_EINVAL;
    }
    *out = nullptr;
    pic_pif* p = new (std::nothrow) pic_pif();
    if (!p) return PIC_ENOMEM;
    p->n = n;
    p->M = 2 * n;
    p->w = width_of(eps);
    p->L = length;
    p->eps = eps;
    p->beta = 2.30 * p->w;
    p->inv_hf = (double)p->M / length;
    p->stream = (cudaStream_t)stream;
    const Layout o = layout(n, np_max, p->w);
    if (bytes < o.total) {
        snprintf(g_err, sizeof(g_err), "workspace %zu bytes < %zu", bytes, o.total);
        delete p;
        return PIC_ENOMEM;
    }
    char* b = (char*)workspace;
    p->G = (double2*)(b + o.G);
    p->A = (double2*)(b + o.A);
    p->Bz = (double2*)(b + o.Bz);
    p->dinv = (double*)(b + o.dinv);
    p->partials = (double*)(b + o.partials);
    p->energy = (double*)(b + o.energy);
    p->hist = (double*)(b + o.hist);
    p->hist_slot = -1;
    p->tw = (double2*)(b + o.tw);
    p->nb = p->M / kB;
    {
        const char* e = getenv("PIC_PIF_BINNED");
        const bool use = (np_max > 0 && binnable(n, p->w)) && !(e && e[0] == '0');
        const char* si = getenv("PIC_PIF_SPLIT_INTERP");
        p->split_interp = si && si[0] == '1';
        p->np_max = use ? np_max : 0;
        p->bcnt = use ? (uint32_t*)(b + o.bcnt) : nullptr;
        p->boffs = use ? (uint32_t*)(b + o.boffs) : nullptr;
        p->bcur = use ? (uint32_t*)(b + o.bcur) : nullptr;
        p->perm = use ? (uint32_t*)(b + o.perm) : nullptr;
        p->G2 = use ? (double2*)(b + o.G2) : nullptr;
        p->scan_tmp = use ? (void*)(b + o.scan) : nullptr;
        const int64_t nbins = (int64_t)p->nb * p->nb * p->nb;
        p->scan_bytes = use ? scan_tmp_bytes(nbins) : 0;
        p->pmask = use ? (uint32_t*)(b + o.pmask) : nullptr;
        p->lmask = use ? p->pmask + p->M : nullptr;
    }
    {   // twiddles of the fine-grid FFT: W_M^m = exp(-2 pi i m / M), m < M
        double2* tw = (double2*)std::malloc(sizeof(double2) * p->M);
        if (!tw) { delete p; return PIC_ENOMEM; }
        for (int m = 0; m < p->M; ++m) {
            const double a = 2.0 * M_PI * (double)m / (double)p->M;
            tw[m] = make_double2(std::cos(a), -std::sin(a));
        }
        const cudaError_t e = cudaMemcpy(p->tw, tw, sizeof(double2) * p->M, cudaMemcpyHostToDevice);
        std::free(tw);
        if (e != cudaSuccess) {
            snprintf(g_err, sizeof(g_err), "twiddle upload: %s", cudaGetErrorString(e));
            delete p;
            return PIC_ECUDA;
        }
    }
    for (auto& e : p->ev) cudaEventCreate(&e);
    k_psihat<<<1, 256, 0, p->stream>>>(n, p->M, p->w, p->beta, p->dinv);
    if (cudaGetLastError() != cudaSuccess) {
        snprintf(g_err, sizeof(g_err), "k_psihat launch failed");
        pic_pif_free(p);
        return PIC_ECUDA;
    }
    *out = p;
    return PIC_OK;
}

pic_status pic_nufft_type1(pic_pif* p, int64_t np, const double* x, const double* f, double* fhat) {
    PIF_CHECK(p);
    if (np < 0 || (np > 0 && (!x || !f)) || !fhat) return PIC_EINVAL;
    if (pic_status s = bin(p, np, x)) return s;
    if (pic_status s = spread(p, np, x, f)) return s;
    if (pic_status s = fft(p, kForward)) return s;
    {
        Stage t(p, PIC_PIF_MODES);
        const int64_t nm = (int64_t)p->n * p->n * p->n;
        k_select<<<stream_grid(nm), kThreads, 0, p->stream>>>(p->n, p->M, p->G, p->dinv, (double2*)fhat);
        PIF_LAUNCHED(p);
        if (p->comm &&
            ncclAllReduce(fhat, fhat, 2 * (size_t)nm, ncclDouble, ncclSum, p->comm, p->stream) != ncclSuccess) {
            snprintf(p->err, sizeof(p->err), "ncclAllReduce of the type-1 sums failed");
            p->poisoned = true;
            return PIC_ENCCL;
        }
    }
    return flush_timing(p);
}

pic_status pic_nufft_type2(pic_pif* p, int64_t np, const double* x, const double* fhat, double* out) {
    PIF_CHECK(p);
    if (np < 0 || (np > 0 && (!x || !out)) || !fhat) return PIC_EINVAL;
    if (pic_status s = bin(p, np, x)) return s;
    if (pic_status s = fill(p, (const double2*)fhat)) return s;
    if (pic_status s = fft(p, kInverse)) return s;
    if (pic_status s = interp(p, np, x, out, out + 1, 2, 1.0)) return s;
    return flush_timing(p);
}

}  // extern "C"

namespace {

pic_status solve_core(pic_pif* p, int64_t np, const double* x, const double* q, double* E) {
    if (pic_status s = bin(p, np, x)) return s;                             // sort into bins
    if (pic_status s = spread(p, np, x, q)) return s;                       // C
    if (pic_status s = fft(p, kForward)) return s;                     // F
    {
        Stage t(p, PIC_PIF_MODES);                                          // chi, D, Poisson
        const double kunit = 2.0 * M_PI / p->L;
        if (p->comm) {   // decomposed: this rank's rho^ (chi, D), summed over the ranks, then Poisson
            const int64_t nm = (int64_t)p->n * p->n * p->n;
            k_select<<<stream_grid(nm), kThreads, 0, p->stream>>>(p->n, p->M, p->G, p->dinv, p->A);
            PIF_LAUNCHED(p);
            if (ncclAllReduce(p->A, p->A, 2 * (size_t)nm, ncclDouble, ncclSum, p->comm, p->stream) != ncclSuccess) {
                snprintf(p->err, sizeof(p->err), "ncclAllReduce of the modes failed");
                p->poisoned = true;
                return PIC_ENCCL;
            }
            k_pif_field<<<kModeBlocks, kThreads, 0, p->stream>>>(p->n, kunit, p->A, p->Bz, p->partials);
        } else {
            k_pif_modes<<<kModeBlocks, kThreads, 0, p->stream>>>(p->n, p->M, kunit, p->G, p->dinv, p->A, p->Bz,
                                                                  p->partials);
        }
        k_energy<<<1, 32, 0, p->stream>>>(kModeBlocks, p->partials, 0.5 / (p->L * p->L * p->L), p->energy,
                                          p->hist_slot >= 0 ? p->hist + p->hist_slot : nullptr);
        PIF_LAUNCHED(p);
    }
    const double sc = 1.0 / (p->L * p->L * p->L);                           // D#35
    if (p->binned && p->G2 && !p->split_interp) {                          // one gather pass
        if (pic_status s = fill(p, p->A)) return s;                         // E_x + i E_y -> G
        if (pic_status s = fft(p, kInverse)) return s;
        if (pic_status s = fill(p, p->Bz, p->G2)) return s;                 // E_z -> G2
        if (pic_status s = fft(p, kInverse, p->G2)) return s;
        Stage t(p, PIC_PIF_INTERP);
        PIF_W_SWITCH_SMALL(p->w, interp3_tiled_w, p, np, x, E, sc);
        PIF_LAUNCHED(p);
        return PIC_OK;
    }
    if (pic_status s = fill(p, p->A)) return s;                             // E_x + i E_y
    if (pic_status s = fft(p, kInverse)) return s;
    if (pic_status s = interp(p, np, x, E, E + np, 1, sc)) return s;
    if (pic_status s = fill(p, p->Bz)) return s;                            // E_z
    if (pic_status s = fft(p, kInverse)) return s;
    return interp(p, np, x, E + 2 * np, nullptr, 1, sc);
}

}  // namespace

extern "C" {

pic_status pic_pif_solve(pic_pif* p, int64_t np, const double* x, const double* q, double* E, double* energy) {
    PIF_CHECK(p);
    if (np < 0 || (np > 0 && (!x || !q || !E))) return PIC_EINVAL;
    p->hist_slot = -1;
    if (pic_status s = solve_core(p, np, x, q, E)) return s;
    if (energy) {
        PIF_CUDA(p, cudaMemcpyAsync(energy, p->energy, 3 * sizeof(double), cudaMemcpyDeviceToHost, p->stream));
        PIF_CUDA(p, cudaStreamSynchronize(p->stream));
        for (int d = 0; d < 3; ++d)
            if (!std::isfinite(energy[d])) {
                snprintf(p->err, sizeof(p->err), "PIF field energy %d is not finite", d);
                return PIC_ENONFINITE;
            }
    }
    return flush_timing(p);
}

pic_status pic_pif_step(pic_pif* p, int64_t np, double* x, double* v, const double* q, double* E, double qm,
                        double dt, int32_t nsteps, double* ex_energy) {
    PIF_CHECK(p);
    if (np < 0 || (np > 0 && (!x || !v || !q || !E)) || nsteps < 1 || nsteps > kMaxSteps) return PIC_EINVAL;
    const double qm_dt = qm * dt;
    for (int s = 0; s < nsteps; ++s) {
        p->hist_slot = s;
        pic_status st = solve_core(p, np, x, q, E);
        p->hist_slot = -1;
        if (st) return st;
        {
            Stage t(p, PIC_PIF_PUSH);
            if (np > 0) k_pif_push<<<particle_grid(np), kThreads, 0, p->stream>>>(np, x, v, E, qm_dt, dt, p->L);
            PIF_LAUNCHED(p);
        }
        // with timing on, collect every step's events (the pool holds 256 event pairs, so a
        // long call would otherwise drop the later steps' stage times)
        if (p->timing) PIC_TRY_PIF(flush_timing(p));
    }
    if (ex_energy) {
        PIF_CUDA(p, cudaMemcpyAsync(ex_energy, p->hist, nsteps * sizeof(double), cudaMemcpyDeviceToHost,
                                    p->stream));
        PIF_CUDA(p, cudaStreamSynchronize(p->stream));
        for (int s = 0; s < nsteps; ++s)
            if (!std::isfinite(ex_energy[s])) {
                snprintf(p->err, sizeof(p->err), "PIF field energy of step %d is not finite", s);
                return PIC_ENONFINITE;
            }
    }
    return flush_timing(p);
}

pic_status pic_pif_set_timing(pic_pif* p, int32_t enable) {
    PIF_CHECK(p);
    p->timing = enable != 0;
    p->nev = 0;
    for (int s = 0; s < PIC_PIF_NSTAGES; ++s) {
        p->ms[s] = 0.0;
        p->launches[s] = 0;
    }
    return PIC_OK;
}

pic_status pic_pif_get_timings(pic_pif* p, double* ms, int64_t* launches) {
    PIF_CHECK(p);
    for (int s = 0; s < PIC_PIF_NSTAGES; ++s) {
        if (ms) ms[s] = p->ms[s];
        if (launches) launches[s] = p->launches[s];
    }
    return PIC_OK;
}

pic_status pic_pif_window(pic_pif* p, int32_t* w, int32_t* m) {
    if (!p) return PIC_EINVAL;
    if (w) *w = p->w;
    if (m) *m = p->M;
    return PIC_OK;
}

pic_status pic_pif_attach_nccl(pic_pif* p, int32_t rank, int32_t nranks, const uint8_t* nccl_id) {
    PIF_CHECK(p);
    if (p->comm || nranks < 1 || rank < 0 || rank >= nranks || (nranks > 1 && !nccl_id)) return PIC_EINVAL;
    if (nranks == 1) return PIC_OK;
    ncclUniqueId u;
    std::memcpy(&u, nccl_id, sizeof(u));
    const ncclResult_t r = ncclCommInitRank(&p->comm, nranks, u, rank);
    if (r != ncclSuccess) {
        snprintf(p->err, sizeof(p->err), "ncclCommInitRank: %s", ncclGetErrorString(r));
        p->comm = nullptr;
        return PIC_ENCCL;
    }
    p->nranks = nranks;
    return PIC_OK;
}

const char* pic_pif_last_error(const pic_pif* p) { return p ? p->err : g_err; }

void pic_pif_free(pic_pif* p) {
    if (!p) return;
    if (p->stream) cudaStreamSynchronize(p->stream);
    if (p->comm) ncclCommDestroy(p->comm);
    for (auto& e : p->ev)
        if (e) cudaEventDestroy(e);
    delete p;
}

}  // extern "C"
