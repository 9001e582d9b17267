// fem_kernels.cu -- the matrix-free Q1 FEM Poisson solve of the PIC step (SURVEY
// §8(f) NEXT-4; P:183-195 first-order Lagrange elements, matrix-free operator, plain
// CG; P:226 tol 1e-4; P:260 warm start; reading D#33).
//
// On the uniform periodic hexahedral mesh the element loop sum_e scatter(A^e gather_e x)
// with the trilinear element stiffness (1/3 on the diagonal, 0 for edge neighbours,
// -1/12 for face-diagonal and opposite vertices, times h) assembles to one 27-point
// stencil: centre 8h/3, face neighbours 0, edge neighbours -h/6, corner neighbours
// -h/12.  That is what a GPU should apply: each node gathers its 26 neighbours once
// (no atomics, no colouring, no per-element conditionals -- the paper's GPU concern,
// P:321) and the result equals the element loop up to summation order.
//
// Fields are natural [zl][y][x] grids of the slab; planes -1 and nzl come from the
// neighbour slabs (P > 1, peer memory) or wrap (P = 1).  A thread owns four
// consecutive nodes of a row (256-bit rows) and a CTA walks a chunk of planes for a
// block of rows (z-march: the stencil's zl +- 1 rows are L1/L2 hits).
#include <cstdlib>

#include "kernels.h"

namespace pic {
namespace {

constexpr int kFT = 256;

struct FNbr {
    const double* own;
    const double* below;
    const double* above;
};
struct R6 {
    double v[6];   // nodes x - 1 .. x + 4 of a row
};

__device__ __forceinline__ const double* frow(const Geom& g, const FNbr& f, int zl, int y) {
    const double* b = f.own;
    if (zl < 0) { b = f.below; zl += g.nzl; }
    else if (zl >= g.nzl) { b = f.above; zl -= g.nzl; }
    return b + ((int64_t)zl * g.n + y) * g.n;
}
__device__ __forceinline__ void ld4f(const double* p, double* o) {
    asm volatile("ld.global.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(o[0]), "=d"(o[1]), "=d"(o[2]), "=d"(o[3]) : "l"(p));
}
__device__ __forceinline__ void st4f(double* p, const double* v) {
    asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(v[0]), "d"(v[1]), "d"(v[2]), "d"(v[3])
                 : "memory");
}
__device__ __forceinline__ R6 ldrow6(const Geom& g, const FNbr& f, int zl, int y, int x) {
    const double* r = frow(g, f, zl, y);
    R6 a;
    ld4f(r + x, a.v + 1);
    a.v[0] = r[(x - 1) & g.nmask];
    a.v[5] = r[(x + 4) & g.nmask];
    return a;
}

struct FMarch {
    int y, x, z0, z1;
    bool on;
};
__device__ __forceinline__ FMarch fmarch(const Geom& g, int cz) {
    const int ipr = g.n >> 2;                          // 4-node items per row
    const int R = min(kFT / ipr, g.n);                 // rows per CTA
    const int nyb = g.n / R;
    FMarch m;
    const int t = threadIdx.x, rr = t / ipr;
    m.on = rr < R;
    m.x = 4 * (t - rr * ipr);
    m.y = (blockIdx.x % nyb) * R + rr;
    m.z0 = (blockIdx.x / nyb) * cz;
    m.z1 = min(m.z0 + cz, g.nzl);
    return m;
}

__device__ __forceinline__ void fblock_partials(double* v, int nv, double* partials) {
    __shared__ double red[3][kFT / 32];
    for (int k = 0; k < nv; ++k) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
        if ((threadIdx.x & 31) == 0) red[k][threadIdx.x >> 5] = v[k];
    }
    __syncthreads();
    if (threadIdx.x < nv) {
        double s = 0.0;
        for (int w = 0; w < kFT / 32; ++w) s += red[threadIdx.x][w];
        partials[(int64_t)threadIdx.x * gridDim.x + blockIdx.x] = s;
    }
}

// The 27-point Q1 stiffness at four nodes (x .. x+3) of row (y, zl); pf (nullable):
// the operand is f + beta pf (formed per loaded value).  out = A f, val = f at the nodes.
__device__ __forceinline__ void apply_q1(const Geom& g, const FNbr& f, const FNbr* pf, double beta, int zl, int y,
                                         int x, double c0, double c2, double c3, double out[4], double val[4]) {
    double s2[4] = {0.0, 0.0, 0.0, 0.0}, s3[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int dz = -1; dz <= 1; ++dz)
#pragma unroll
        for (int dy = -1; dy <= 1; ++dy) {
            const int yy = (y + dy) & g.nmask, zz = zl + dz;
            R6 a = ldrow6(g, f, zz, yy, x);
            if (pf) {
                const R6 b = ldrow6(g, *pf, zz, yy, x);
#pragma unroll
                for (int k = 0; k < 6; ++k) a.v[k] = __dadd_rn(a.v[k], __dmul_rn(beta, b.v[k]));
            }
            const int mr = (dy != 0) + (dz != 0);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const double side = __dadd_rn(a.v[k], a.v[k + 2]);   // x - 1, x + 1
                if (mr == 0) val[k] = a.v[k + 1];
                else if (mr == 1) s2[k] = __dadd_rn(s2[k], side);
                else {
                    s2[k] = __dadd_rn(s2[k], a.v[k + 1]);
                    s3[k] = __dadd_rn(s3[k], side);
                }
            }
        }
#pragma unroll
    for (int k = 0; k < 4; ++k)
        out[k] = __dsub_rn(__dsub_rn(__dmul_rn(c0, val[k]), __dmul_rn(c2, s2[k])), __dmul_rn(c3, s3[k]));
}

// sum_m h^3 dscale raw_m (the load before its mean is removed), partial per CTA.
__global__ void __launch_bounds__(kFT) k_fem_load_sum(Geom g, const double* __restrict__ raw, double dscale,
                                                      double h3, int cz, double* __restrict__ partials) {
    const FMarch m = fmarch(g, cz);
    double acc = 0.0;
    for (int zl = m.z0; m.on && zl < m.z1; ++zl) {
        double v[4];
        ld4f(raw + ((int64_t)zl * g.n + m.y) * g.rp + m.x, v);
#pragma unroll
        for (int k = 0; k < 4; ++k) acc += __dmul_rn(h3, __dmul_rn(dscale, v[k]));
    }
    fblock_partials(&acc, 1, partials);
}

// r = (h^3 rho - mean) - A x; partials (b, b), (r, r).
__global__ void __launch_bounds__(kFT) k_fem_resid0(Geom g, const double* __restrict__ raw, double dscale,
                                                    double h3, const double* __restrict__ sc, double nn, FNbr x,
                                                    double* __restrict__ r, double c0, double c2, double c3,
                                                    int cz, double* __restrict__ partials) {
    const FMarch m = fmarch(g, cz);
    const double mean = sc[0] / nn;
    double acc[2] = {0.0, 0.0};
    for (int zl = m.z0; m.on && zl < m.z1; ++zl) {
        double v[4], ax[4], xv[4], rv[4];
        ld4f(raw + ((int64_t)zl * g.n + m.y) * g.rp + m.x, v);
        apply_q1(g, x, nullptr, 0.0, zl, m.y, m.x, c0, c2, c3, ax, xv);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const double b = __dsub_rn(__dmul_rn(h3, __dmul_rn(dscale, v[k])), mean);
            rv[k] = __dsub_rn(b, ax[k]);
            acc[0] = fma(b, b, acc[0]);
            acc[1] = fma(rv[k], rv[k], acc[1]);
        }
        st4f(r + ((int64_t)zl * g.n + m.y) * g.n + m.x, rv);
    }
    fblock_partials(acc, 2, partials);
}

// p' = r + beta p (first: r), q = A p', partial (p', q); beta = sc[2] / sc[4].
// STORE = false: the operand is already p' (formed by k_fem_paxpy), only q is written.
template <bool FIRST, bool STORE = true>
__global__ void __launch_bounds__(kFT) k_fem_matvec(Geom g, FNbr r, FNbr p, double* __restrict__ pout,
                                                    double* __restrict__ q, const double* __restrict__ sc,
                                                    double c0, double c2, double c3, int cz,
                                                    double* __restrict__ partials) {
    const FMarch m = fmarch(g, cz);
    const double beta = FIRST ? 0.0 : sc[2] / sc[4];
    double acc = 0.0;
    for (int zl = m.z0; m.on && zl < m.z1; ++zl) {
        double av[4], pv[4];
        apply_q1(g, r, FIRST ? nullptr : &p, beta, zl, m.y, m.x, c0, c2, c3, av, pv);
        const int64_t o = ((int64_t)zl * g.n + m.y) * g.n + m.x;
        if (STORE) st4f(pout + o, pv);
        st4f(q + o, av);
#pragma unroll
        for (int k = 0; k < 4; ++k) acc = fma(pv[k], av[k], acc);
    }
    fblock_partials(&acc, 1, partials);
    if (g.P > 1) __threadfence_system();
}

// p' = r + beta p, streaming (the split matvec: the stencil then reads one field).
__global__ void __launch_bounds__(kFT) k_fem_paxpy(int64_t n4, const double* __restrict__ r,
                                                   const double* __restrict__ p, double* __restrict__ pout,
                                                   const double* __restrict__ sc) {
    const double beta = sc[2] / sc[4];
    for (int64_t i = (int64_t)blockIdx.x * kFT + threadIdx.x; i < n4; i += (int64_t)gridDim.x * kFT) {
        double rv[4], pv[4];
        ld4f(r + 4 * i, rv);
        ld4f(p + 4 * i, pv);
#pragma unroll
        for (int k = 0; k < 4; ++k) pv[k] = __dadd_rn(rv[k], __dmul_rn(beta, pv[k]));
        st4f(pout + 4 * i, pv);
    }
}

// x += alpha p ; r -= alpha q ; partial (r, r); alpha = sc[2] / sc[5].
__global__ void __launch_bounds__(kFT) k_fem_update(int64_t n4, int sys_fence, double* __restrict__ x,
                                                    const double* __restrict__ p, double* __restrict__ r,
                                                    const double* __restrict__ q, const double* __restrict__ sc,
                                                    double* __restrict__ partials) {
    const double alpha = sc[2] / sc[5];
    double acc = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * kFT + threadIdx.x; i < n4; i += (int64_t)gridDim.x * kFT) {
        double pv[4], qv[4], xv[4], rv[4];
        ld4f(p + 4 * i, pv);
        ld4f(q + 4 * i, qv);
        ld4f(x + 4 * i, xv);
        ld4f(r + 4 * i, rv);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            xv[k] = __dadd_rn(xv[k], __dmul_rn(alpha, pv[k]));
            rv[k] = __dsub_rn(rv[k], __dmul_rn(alpha, qv[k]));
            acc = fma(rv[k], rv[k], acc);
        }
        st4f(x + 4 * i, xv);
        st4f(r + 4 * i, rv);
    }
    fblock_partials(&acc, 1, partials);
    if (sys_fence) __threadfence_system();
}

// E = -grad_h phi (central differences, D#30) -> E4 (+ plane 0 into halo), E_d^2 partials.
__global__ void __launch_bounds__(kFT) k_fem_gradient(Geom g, FNbr x, double* __restrict__ E4, double* halo, int cz,
                                                      double* __restrict__ partials) {
    const FMarch m = fmarch(g, cz);
    const double cc = 0.5 * g.inv_h;
    double e2[3] = {0.0, 0.0, 0.0};
    for (int zl = m.z0; m.on && zl < m.z1; ++zl) {
        const R6 c = ldrow6(g, x, zl, m.y, m.x);
        double ym[4], yp[4], zm[4], zp[4];
        ld4f(frow(g, x, zl, (m.y - 1) & g.nmask) + m.x, ym);
        ld4f(frow(g, x, zl, (m.y + 1) & g.nmask) + m.x, yp);
        ld4f(frow(g, x, zl - 1, m.y) + m.x, zm);
        ld4f(frow(g, x, zl + 1, m.y) + m.x, zp);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const double ex = __dmul_rn(__dsub_rn(c.v[k], c.v[k + 2]), cc);
            const double ey = __dmul_rn(__dsub_rn(ym[k], yp[k]), cc);
            const double ez = __dmul_rn(__dsub_rn(zm[k], zp[k]), cc);
            const int64_t nd = 4 * (((int64_t)zl * g.n + m.y) * g.n + m.x + k);
            asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(E4 + nd), "d"(ex), "d"(ey), "d"(ez),
                         "d"(0.0) : "memory");
            if (halo && zl == 0)
                asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(halo + nd), "d"(ex), "d"(ey),
                             "d"(ez), "d"(0.0) : "memory");
            e2[0] = fma(ex, ex, e2[0]);
            e2[1] = fma(ey, ey, e2[1]);
            e2[2] = fma(ez, ez, e2[2]);
        }
    }
    fblock_partials(e2, 3, partials);
    if (halo && g.P > 1) __threadfence_system();
}

// One CTA, fixed order (deterministic): out[k] = sum of partials[k][...]; save: out[0]
// is first copied to *save; energy: out = (W_x, W).
__global__ void __launch_bounds__(1024) k_fem_reduce(Geom g, const double* __restrict__ partials, int nparts,
                                                     int ncomp, double* out, double* save, int energy) {
    __shared__ double red[3][32];
    double s[3] = {0.0, 0.0, 0.0};
    for (int k = 0; k < ncomp; ++k)
        for (int i = threadIdx.x; i < nparts; i += blockDim.x) s[k] += partials[(int64_t)k * nparts + i];
    for (int k = 0; k < ncomp; ++k) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s[k] += __shfl_xor_sync(0xffffffffu, s[k], o);
        if ((threadIdx.x & 31) == 0) red[k][threadIdx.x >> 5] = s[k];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double t[3] = {0.0, 0.0, 0.0};
        for (int k = 0; k < ncomp; ++k)
            for (int w = 0; w < (int)(blockDim.x / 32); ++w) t[k] += red[k][w];
        if (save) *save = out[0];
        if (energy) {
            const double h = g.L / (double)g.n;
            const double h3 = (h * h) * h;
            out[0] = 0.5 * h3 * t[0];
            out[1] = 0.5 * h3 * (t[0] + t[1] + t[2]);
        } else {
            for (int k = 0; k < ncomp; ++k) out[k] = t[k];
        }
    }
}

// (row blocks) x (plane chunks of cz), ~2048 CTAs (<= 4095: the partials buffer).
unsigned fmarch_grid(const Geom& g, int* cz) {
    const int ipr = g.n >> 2, R = std::min(kFT / ipr, g.n), nyb = g.n / R;
    int c = 1;
    while (c < g.nzl && (int64_t)nyb * (g.nzl / (2 * c)) >= 2048) c *= 2;
    *cz = c;
    return (unsigned)(nyb * ((g.nzl + c - 1) / c));
}

struct Q1 {
    double c0, c2, c3;
};
Q1 q1_coeffs(const Geom& g) {
    const double h = g.L / (double)g.n;
    return Q1{(8.0 / 3.0) * h, h / 6.0, h / 12.0};
}
FNbr fn(const PcgNbr& a) { return FNbr{a.own, a.below, a.above}; }

}  // namespace

void launch_fem_load_sum(const Geom& g, const double* raw, double dscale, double* partials, double* sc,
                         cudaStream_t s) {
    int cz = 1;
    const unsigned grid = fmarch_grid(g, &cz);
    const double h = g.L / (double)g.n;
    k_fem_load_sum<<<grid, kFT, 0, s>>>(g, raw, dscale, (h * h) * h, cz, partials);
    k_fem_reduce<<<1, 1024, 0, s>>>(g, partials, (int)grid, 1, sc, nullptr, 0);
}

void launch_fem_resid0(const Geom& g, const double* raw, double dscale, double* sc, double nn, PcgNbr x,
                       double* r, double* partials, cudaStream_t s) {
    int cz = 1;
    const unsigned grid = fmarch_grid(g, &cz);
    const double h = g.L / (double)g.n;
    const Q1 q = q1_coeffs(g);
    k_fem_resid0<<<grid, kFT, 0, s>>>(g, raw, dscale, (h * h) * h, sc, nn, fn(x), r, q.c0, q.c2, q.c3, cz, partials);
    k_fem_reduce<<<1, 1024, 0, s>>>(g, partials, (int)grid, 2, sc + 1, nullptr, 0);
}

void launch_fem_matvec(const Geom& g, bool first, PcgNbr r, PcgNbr p, double* pout, double* q, double* sc,
                       double* partials, cudaStream_t s) {
    int cz = 1;
    const unsigned grid = fmarch_grid(g, &cz);
    const Q1 c = q1_coeffs(g);
    if (first) k_fem_matvec<true><<<grid, kFT, 0, s>>>(g, fn(r), fn(p), pout, q, sc, c.c0, c.c2, c.c3, cz, partials);
    else k_fem_matvec<false><<<grid, kFT, 0, s>>>(g, fn(r), fn(p), pout, q, sc, c.c0, c.c2, c.c3, cz, partials);
    k_fem_reduce<<<1, 1024, 0, s>>>(g, partials, (int)grid, 1, sc + 5, nullptr, 0);
}

bool fem_split() {
    const char* e = getenv("PIC_FEM_SPLIT");
    return !(e && e[0] == '0');
}

void launch_fem_paxpy(const Geom& g, const double* r, const double* p, double* pout, const double* sc,
                      cudaStream_t s) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t n4 = (int64_t)g.n * g.n * g.nzl / 4;
    const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n4 + kFT - 1) / kFT, (int64_t)sms * 8));
    k_fem_paxpy<<<grid, kFT, 0, s>>>(n4, r, p, pout, sc);
}

void launch_fem_stencil(const Geom& g, PcgNbr p, double* q, double* sc, double* partials, cudaStream_t s) {
    int cz = 1;
    const unsigned grid = fmarch_grid(g, &cz);
    const Q1 c = q1_coeffs(g);
    k_fem_matvec<true, false><<<grid, kFT, 0, s>>>(g, fn(p), fn(p), nullptr, q, sc, c.c0, c.c2, c.c3, cz, partials);
    k_fem_reduce<<<1, 1024, 0, s>>>(g, partials, (int)grid, 1, sc + 5, nullptr, 0);
}

void launch_fem_update(const Geom& g, double* x, const double* p, double* r, const double* q, double* sc,
                       double* partials, cudaStream_t s) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t n4 = (int64_t)g.n * g.n * g.nzl / 4;
    const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n4 + kFT - 1) / kFT, (int64_t)sms * 8));
    k_fem_update<<<grid, kFT, 0, s>>>(n4, g.P > 1, x, p, r, q, sc, partials);
    k_fem_reduce<<<1, 1024, 0, s>>>(g, partials, (int)grid, 1, sc + 2, sc + 4, 0);
}

void launch_fem_gradient(const Geom& g, PcgNbr x, double* E4, double* halo, double* partials, double* energies,
                         cudaStream_t s) {
    int cz = 1;
    const unsigned grid = fmarch_grid(g, &cz);
    k_fem_gradient<<<grid, kFT, 0, s>>>(g, fn(x), E4, halo, cz, partials);
    k_fem_reduce<<<1, 1024, 0, s>>>(g, partials, (int)grid, 3, energies, nullptr, 1);
}

}  // namespace pic
