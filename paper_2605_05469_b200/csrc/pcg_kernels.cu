// pcg_kernels.cu -- the FD-PCG Poisson solve of the PIC step (BJ config 5):
// -Delta_h phi = rho - mean(rho) by SSOR-preconditioned CG, E = -grad_h phi
// (P:179-181 second-order finite differences, matrix-free CG; P:260 SSOR with
// four inner and two outer iterations and damping pi/2, warm start
// tolerance 1e-4; readings D#26-D#31).
//
// Layout ("colour-split"): a field F of the slab is stored as two half grids
// F[c][zl][y][j], c = (x + y + z) mod 2 (red 0, black 1), j = x / 2 -- so the
// node x of row (y, zl) is element x >> 1 of colour (x + y + zl) & 1 (z0 is even,
// so local and global z parity agree).  A red/black half-sweep then streams its
// own colour and reads the other one: every access is a coalesced run, and a
// half-sweep moves 16 B per node (own z r/w, own r, other z) instead of touching
// both colours of every sector.  The six neighbours of a node all have the other
// colour; in that colour they sit at elements j - 1 + o and j + o of the same row
// (o = x & 1) and at element j of the rows y +- 1 and planes zl +- 1.  Plane -1 and
// plane nzl are the planes of the slabs below / above (P = 1: this slab, periodic),
// read straight from the peer's buffer over NVLink at P > 1.
//
// Dot products: grid-stride kernels with a fixed grid leave one partial per CTA;
// k_pcg_reduce sums them in a fixed order (deterministic run to run).
#include "kernels.h"

namespace pic {
namespace {

constexpr int kPT = 256;   // threads per CTA

// Element j of colour c in row (y, zl) of a colour-split field.
__device__ __forceinline__ int64_t sidx(const Geom& g, int c, int zl, int y, int j) {
    return (((int64_t)c * g.nzl + zl) * g.n + y) * (g.n >> 1) + j;
}

// The same with zl in [-1, nzl]: planes outside the slab come from the field of
// the rank below / above (P = 1: this one, periodic).
struct Nbr {
    const double* own;
    const double* below;
    const double* above;
};
__device__ __forceinline__ double ldz(const Geom& g, const Nbr& f, int c, int zl, int y, int j) {
    const double* b = f.own;
    if (zl < 0) { b = f.below; zl += g.nzl; }
    else if (zl >= g.nzl) { b = f.above; zl -= g.nzl; }
    return b[sidx(g, c, zl, y, j)];
}
__device__ __forceinline__ double2 ldz2(const Geom& g, const Nbr& f, int c, int zl, int y, int j) {
    const double* b = f.own;
    if (zl < 0) { b = f.below; zl += g.nzl; }
    else if (zl >= g.nzl) { b = f.above; zl -= g.nzl; }
    return *reinterpret_cast<const double2*>(b + sidx(g, c, zl, y, j));
}

// Neighbour sum in the oracle's order: ((xm + xp) + (ym + yp)) + (zm + zp).
__device__ __forceinline__ double nsum(double xm, double xp, double ym, double yp, double zm, double zp) {
    return __dadd_rn(__dadd_rn(__dadd_rn(xm, xp), __dadd_rn(ym, yp)), __dadd_rn(zm, zp));
}

__device__ __forceinline__ void block_partials(double* v, int nv, double* partials) {
    __shared__ double red[4][kPT / 32];
    for (int k = 0; k < nv; ++k) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
        if ((threadIdx.x & 31) == 0) red[k][threadIdx.x >> 5] = v[k];
    }
    __syncthreads();
    if (threadIdx.x < nv) {
        double s = 0.0;
        for (int w = 0; w < kPT / 32; ++w) s += red[threadIdx.x][w];
        partials[(int64_t)threadIdx.x * gridDim.x + blockIdx.x] = s;
    }
}

// Row decomposition of a pair index p (pairs of elements j, j+1 of one colour row;
// or natural node pairs x = 2j, 2j + 1 of one row).
struct PairPos {
    int zl, y, j;
};
__device__ __forceinline__ PairPos pair_pos(const Geom& g, int64_t p) {
    const int hp = g.n >> 2;                 // pairs per row
    const int64_t row = p / hp;
    PairPos q;
    q.j = 2 * (int)(p - row * hp);
    q.y = (int)(row & g.nmask);
    q.zl = (int)(row / g.n);
    return q;
}

// ------------------------------------------------------------ SOR sweep -----
// One SOR half-sweep of colour c (D#28): z_m <- (1 - omega) z_m + (omega/6)(h^2 r_m + nb).
// MODE 0: general; 1: z of colour c is zero (its first update); 2: z is zero
// everywhere (the first half-sweep of M^-1).  DOT: also the partial of (r, z) over
// both colours (the last half-sweep of M^-1).  Thread = two elements j, j+1.
template <int MODE, bool DOT>
__global__ void __launch_bounds__(kPT) k_sor(Geom g, int c, const double* __restrict__ r, Nbr z, double* zout,
                                             double c1, double c2, double h2, double* __restrict__ partials) {
    const int hn = g.n >> 1, oc = c ^ 1;
    const int64_t npair = (int64_t)g.n * g.nzl * (g.n >> 2);
    double acc = 0.0;
    for (int64_t p = (int64_t)blockIdx.x * kPT + threadIdx.x; p < npair; p += (int64_t)gridDim.x * kPT) {
        const PairPos q = pair_pos(g, p);
        const int o = (q.y + q.zl + c) & 1;          // x of element j is 2j + o
        const int64_t me = sidx(g, c, q.zl, q.y, q.j);
        const double2 rv = *reinterpret_cast<const double2*>(r + me);
        double2 zn;
        double2 m = make_double2(0.0, 0.0);
        if (MODE == 2) {
            zn.x = __dmul_rn(c2, __dmul_rn(h2, rv.x));
            zn.y = __dmul_rn(c2, __dmul_rn(h2, rv.y));
        } else {
            m = ldz2(g, z, oc, q.zl, q.y, q.j);                       // other colour, j and j+1
            const double e = o ? ldz(g, z, oc, q.zl, q.y, (q.j + 2) & (hn - 1))
                               : ldz(g, z, oc, q.zl, q.y, (q.j - 1) & (hn - 1));
            const double2 ym = ldz2(g, z, oc, q.zl, (q.y - 1) & g.nmask, q.j);
            const double2 yp = ldz2(g, z, oc, q.zl, (q.y + 1) & g.nmask, q.j);
            const double2 zm = ldz2(g, z, oc, q.zl - 1, q.y, q.j);
            const double2 zp = ldz2(g, z, oc, q.zl + 1, q.y, q.j);
            // element j: x-neighbours other[j - 1 + o], other[j + o]; element j + 1: shifted by one
            const double x0m = o ? m.x : e, x0p = o ? m.y : m.x;
            const double x1m = o ? m.y : m.x, x1p = o ? e : m.y;
            const double s0 = nsum(x0m, x0p, ym.x, yp.x, zm.x, zp.x);
            const double s1 = nsum(x1m, x1p, ym.y, yp.y, zm.y, zp.y);
            double2 zo = make_double2(0.0, 0.0);
            if (MODE == 0) zo = *reinterpret_cast<const double2*>(z.own + me);
            zn.x = __dadd_rn(__dmul_rn(c1, zo.x), __dmul_rn(c2, __dadd_rn(__dmul_rn(h2, rv.x), s0)));
            zn.y = __dadd_rn(__dmul_rn(c1, zo.y), __dmul_rn(c2, __dadd_rn(__dmul_rn(h2, rv.y), s1)));
        }
        *reinterpret_cast<double2*>(zout + me) = zn;
        if (DOT) {
            // this colour's pair and the other colour's pair (j, j+1) of the same row
            const double2 ro = *reinterpret_cast<const double2*>(r + sidx(g, oc, q.zl, q.y, q.j));
            acc = fma(rv.x, zn.x, acc);
            acc = fma(rv.y, zn.y, acc);
            acc = fma(ro.x, m.x, acc);
            acc = fma(ro.y, m.y, acc);
        }
    }
    if (DOT) block_partials(&acc, 1, partials);
    if (g.P > 1) __threadfence_system();
}

// ------------------------------------------------------- natural pairs ------
// Values of a field at the nodes x = 2j, 2j+1 of row (y, zl) (zl in [-1, nzl]).
__device__ __forceinline__ double2 ldnat(const Geom& g, const Nbr& f, int zl, int y, int j) {
    const int c0 = (y + zl) & 1;   // colour of x = 2j (zl + nzl has the parity of zl)
    return make_double2(ldz(g, f, c0, zl, y, j), ldz(g, f, c0 ^ 1, zl, y, j));
}
__device__ __forceinline__ void stnat(const Geom& g, double* f, int zl, int y, int j, double2 v) {
    const int c0 = (y + zl) & 1;
    f[sidx(g, c0, zl, y, j)] = v.x;
    f[sidx(g, c0 ^ 1, zl, y, j)] = v.y;
}

// The seven-point neighbourhood of the node pair (2j, 2j+1): left = node 2j - 1,
// right = node 2j + 2, and the pairs of rows y +- 1 and planes zl +- 1.
struct Hood {
    double2 c, ym, yp, zm, zp;
    double left, right;
};
__device__ __forceinline__ Hood ldhood(const Geom& g, const Nbr& f, int zl, int y, int j) {
    const int hn = g.n >> 1, c0 = (y + zl) & 1;
    Hood h;
    h.c = ldnat(g, f, zl, y, j);
    h.left = ldz(g, f, c0 ^ 1, zl, y, (j - 1) & (hn - 1));
    h.right = ldz(g, f, c0, zl, y, (j + 1) & (hn - 1));
    h.ym = ldnat(g, f, zl, (y - 1) & g.nmask, j);
    h.yp = ldnat(g, f, zl, (y + 1) & g.nmask, j);
    h.zm = ldnat(g, f, zl - 1, y, j);
    h.zp = ldnat(g, f, zl + 1, y, j);
    return h;
}
// -Delta_h at the pair (D#26): (6 x - nb) * ih2, nb in the oracle's order.
__device__ __forceinline__ double2 apply_A(const Hood& h, double ih2) {
    const double s0 = nsum(h.left, h.c.y, h.ym.x, h.yp.x, h.zm.x, h.zp.x);
    const double s1 = nsum(h.c.x, h.right, h.ym.y, h.yp.y, h.zm.y, h.zp.y);
    return make_double2(__dmul_rn(__dsub_rn(__dmul_rn(6.0, h.c.x), s0), ih2),
                        __dmul_rn(__dsub_rn(__dmul_rn(6.0, h.c.y), s1), ih2));
}

// sum_m rho_m, rho_m = dscale * raw_m (the raw CIC sums of the pitched rho planes).
__global__ void __launch_bounds__(kPT) k_pcg_rho_sum(Geom g, const double* __restrict__ raw, double dscale,
                                                     double* __restrict__ partials) {
    const int64_t npair = (int64_t)g.n * g.nzl * (g.n >> 2) * 2;   // natural pairs
    const int hq = g.n >> 1;
    double acc = 0.0;
    for (int64_t p = (int64_t)blockIdx.x * kPT + threadIdx.x; p < npair; p += (int64_t)gridDim.x * kPT) {
        const int64_t row = p / hq;
        const int x = 2 * (int)(p - row * hq);
        const double2 v = *reinterpret_cast<const double2*>(raw + row * g.rp + x);
        acc += __dmul_rn(dscale, v.x);
        acc += __dmul_rn(dscale, v.y);
    }
    block_partials(&acc, 1, partials);
}

// r = (rho - mean) - A x (D#27), partials of (b, b) and (r, r).  Thread = natural pair.
__global__ void __launch_bounds__(kPT) k_pcg_resid0(Geom g, const double* __restrict__ raw, double dscale,
                                                    const double* __restrict__ sc, double nn, Nbr x,
                                                    double* __restrict__ r, double ih2,
                                                    double* __restrict__ partials) {
    const int64_t npair = (int64_t)g.n * g.nzl * (g.n >> 1);
    const int hq = g.n >> 1;
    const double mean = sc[0] / nn;
    double acc[2] = {0.0, 0.0};
    for (int64_t p = (int64_t)blockIdx.x * kPT + threadIdx.x; p < npair; p += (int64_t)gridDim.x * kPT) {
        const int64_t row = p / hq;
        const int j = (int)(p - row * hq), y = (int)(row & g.nmask), zl = (int)(row / g.n);
        const double2 v = *reinterpret_cast<const double2*>(raw + row * g.rp + 2 * j);
        const double b0 = __dsub_rn(__dmul_rn(dscale, v.x), mean);
        const double b1 = __dsub_rn(__dmul_rn(dscale, v.y), mean);
        const double2 ax = apply_A(ldhood(g, x, zl, y, j), ih2);
        const double2 rv = make_double2(__dsub_rn(b0, ax.x), __dsub_rn(b1, ax.y));
        stnat(g, r, zl, y, j, rv);
        acc[0] = fma(b0, b0, fma(b1, b1, acc[0]));
        acc[1] = fma(rv.x, rv.x, fma(rv.y, rv.y, acc[1]));
    }
    block_partials(acc, 2, partials);
}

// p' = z + beta p (first: p' = z), q = A p', partial (p', q).  The neighbours' p'
// are formed on the fly from z and p, so p' and q are written once.
template <bool FIRST>
__global__ void __launch_bounds__(kPT) k_pcg_matvec(Geom g, Nbr z, Nbr p, double* __restrict__ pout,
                                                    double* __restrict__ q, const double* __restrict__ sc,
                                                    double ih2, double* __restrict__ partials) {
    const int64_t npair = (int64_t)g.n * g.nzl * (g.n >> 1);
    const int hq = g.n >> 1;
    const double beta = FIRST ? 0.0 : sc[3] / sc[4];
    double acc = 0.0;
    for (int64_t t = (int64_t)blockIdx.x * kPT + threadIdx.x; t < npair; t += (int64_t)gridDim.x * kPT) {
        const int64_t row = t / hq;
        const int j = (int)(t - row * hq), y = (int)(row & g.nmask), zl = (int)(row / g.n);
        Hood h = ldhood(g, z, zl, y, j);
        if (!FIRST) {
            const Hood hp = ldhood(g, p, zl, y, j);
            auto upd = [&](double& a, double b) { a = __dadd_rn(a, __dmul_rn(beta, b)); };
            upd(h.c.x, hp.c.x); upd(h.c.y, hp.c.y);
            upd(h.ym.x, hp.ym.x); upd(h.ym.y, hp.ym.y);
            upd(h.yp.x, hp.yp.x); upd(h.yp.y, hp.yp.y);
            upd(h.zm.x, hp.zm.x); upd(h.zm.y, hp.zm.y);
            upd(h.zp.x, hp.zp.x); upd(h.zp.y, hp.zp.y);
            upd(h.left, hp.left); upd(h.right, hp.right);
        }
        const double2 qv = apply_A(h, ih2);
        stnat(g, pout, zl, y, j, h.c);
        stnat(g, q, zl, y, j, qv);
        acc = fma(h.c.x, qv.x, fma(h.c.y, qv.y, acc));
    }
    block_partials(&acc, 1, partials);
    if (g.P > 1) __threadfence_system();
}

// x += alpha p ; r -= alpha q ; partial (r, r).  alpha = (r, z) / (p, q).
__global__ void __launch_bounds__(kPT) k_pcg_update(int64_t n2, int sys_fence, double2* __restrict__ x,
                                                    const double2* __restrict__ p, double2* __restrict__ r,
                                                    const double2* __restrict__ q, const double* __restrict__ sc,
                                                    double* __restrict__ partials) {
    const double alpha = sc[3] / sc[5];
    double acc = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * kPT + threadIdx.x; i < n2; i += (int64_t)gridDim.x * kPT) {
        const double2 pv = p[i], qv = q[i];
        double2 xv = x[i], rv = r[i];
        xv.x = __dadd_rn(xv.x, __dmul_rn(alpha, pv.x));
        xv.y = __dadd_rn(xv.y, __dmul_rn(alpha, pv.y));
        rv.x = __dsub_rn(rv.x, __dmul_rn(alpha, qv.x));
        rv.y = __dsub_rn(rv.y, __dmul_rn(alpha, qv.y));
        x[i] = xv;
        r[i] = rv;
        acc = fma(rv.x, rv.x, fma(rv.y, rv.y, acc));
    }
    block_partials(&acc, 1, partials);
    if (sys_fence) __threadfence_system();     // x is read by the neighbour slabs
}

__device__ __forceinline__ void st_node4(double* p, double a, double b, double c) {
    asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(0.0)
                 : "memory");
}

// E = -grad_h phi by central differences (D#30) -> E4 node records (+ plane 0 into
// `halo`, the halo plane of the slab below), partials of E_d^2.
__global__ void __launch_bounds__(kPT) k_pcg_gradient(Geom g, Nbr x, double* __restrict__ E4, double* halo,
                                                      double* __restrict__ partials) {
    const int64_t npair = (int64_t)g.n * g.nzl * (g.n >> 1);
    const int hq = g.n >> 1;
    const double cc = 0.5 * g.inv_h;
    double e2[3] = {0.0, 0.0, 0.0};
    for (int64_t t = (int64_t)blockIdx.x * kPT + threadIdx.x; t < npair; t += (int64_t)gridDim.x * kPT) {
        const int64_t row = t / hq;
        const int j = (int)(t - row * hq), y = (int)(row & g.nmask), zl = (int)(row / g.n);
        const Hood h = ldhood(g, x, zl, y, j);
        const double ex0 = __dmul_rn(__dsub_rn(h.left, h.c.y), cc);
        const double ex1 = __dmul_rn(__dsub_rn(h.c.x, h.right), cc);
        const double ey0 = __dmul_rn(__dsub_rn(h.ym.x, h.yp.x), cc);
        const double ey1 = __dmul_rn(__dsub_rn(h.ym.y, h.yp.y), cc);
        const double ez0 = __dmul_rn(__dsub_rn(h.zm.x, h.zp.x), cc);
        const double ez1 = __dmul_rn(__dsub_rn(h.zm.y, h.zp.y), cc);
        const int64_t nd = 4 * (row * g.n + 2 * j);
        st_node4(E4 + nd, ex0, ey0, ez0);
        st_node4(E4 + nd + 4, ex1, ey1, ez1);
        if (halo && zl == 0) {
            st_node4(halo + nd, ex0, ey0, ez0);
            st_node4(halo + nd + 4, ex1, ey1, ez1);
        }
        e2[0] = fma(ex0, ex0, fma(ex1, ex1, e2[0]));
        e2[1] = fma(ey0, ey0, fma(ey1, ey1, e2[1]));
        e2[2] = fma(ez0, ez0, fma(ez1, ez1, e2[2]));
    }
    block_partials(e2, 3, partials);
    if (halo && g.P > 1) __threadfence_system();
}

// One CTA, fixed order: out[k] = sum of partials[k][0..nparts) (k < ncomp).  save:
// out[0] is first copied to *save (rz -> rz_old).  energy: out = (W_x, W) (D#12).
__global__ void __launch_bounds__(1024) k_pcg_reduce(Geom g, const double* __restrict__ partials, int nparts,
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

// Colour-split field -> natural [nzl][n][n] (host transfers of phi).
__global__ void k_pcg_unsplit(Geom g, const double* __restrict__ f, double* __restrict__ out) {
    const int64_t nn = (int64_t)g.n * g.n * g.nzl;
    const int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (m >= nn) return;
    const int x = (int)(m & g.nmask);
    const int64_t row = m / g.n;
    const int y = (int)(row & g.nmask), zl = (int)(row / g.n);
    out[m] = f[sidx(g, (x + y + zl) & 1, zl, y, x >> 1)];
}

unsigned pcg_grid(const Geom& g) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t npair = (int64_t)g.n * g.n * g.nzl / 2;
    const int64_t need = (npair + kPT - 1) / kPT;
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)sms * 8));
}

}  // namespace

void launch_pcg_rho_sum(const Geom& g, const double* raw, double dscale, double* partials, double* sc,
                        cudaStream_t s) {
    const unsigned grid = pcg_grid(g);
    k_pcg_rho_sum<<<grid, kPT, 0, s>>>(g, raw, dscale, partials);
    k_pcg_reduce<<<1, 1024, 0, s>>>(g, partials, (int)grid, 1, sc, nullptr, 0);
}

void launch_pcg_resid0(const Geom& g, const double* raw, double dscale, double* sc, double nn, PcgNbr x,
                       double* r, double* partials, cudaStream_t s) {
    const unsigned grid = pcg_grid(g);
    const double ih2 = g.inv_h * g.inv_h;
    k_pcg_resid0<<<grid, kPT, 0, s>>>(g, raw, dscale, sc, nn, Nbr{x.own, x.below, x.above}, r, ih2, partials);
    k_pcg_reduce<<<1, 1024, 0, s>>>(g, partials, (int)grid, 2, sc + 1, nullptr, 0);
}

void launch_pcg_sor(const Geom& g, int colour, int mode, bool dot, const double* r, PcgNbr z, double omega,
                    double* partials, double* sc, cudaStream_t s) {
    const unsigned grid = pcg_grid(g);
    const double h = g.L / (double)g.n;
    const double h2 = h * h, c1 = 1.0 - omega, c2 = omega / 6.0;
    const Nbr zn{z.own, z.below, z.above};
    double* zo = const_cast<double*>(z.own);
    if (mode == 2) k_sor<2, false><<<grid, kPT, 0, s>>>(g, colour, r, zn, zo, c1, c2, h2, partials);
    else if (mode == 1) k_sor<1, false><<<grid, kPT, 0, s>>>(g, colour, r, zn, zo, c1, c2, h2, partials);
    else if (dot) k_sor<0, true><<<grid, kPT, 0, s>>>(g, colour, r, zn, zo, c1, c2, h2, partials);
    else k_sor<0, false><<<grid, kPT, 0, s>>>(g, colour, r, zn, zo, c1, c2, h2, partials);
    if (dot) k_pcg_reduce<<<1, 1024, 0, s>>>(g, partials, (int)grid, 1, sc + 3, sc + 4, 0);
}

void launch_pcg_matvec(const Geom& g, bool first, PcgNbr z, PcgNbr p, double* pout, double* q, double* sc,
                       double* partials, cudaStream_t s) {
    const unsigned grid = pcg_grid(g);
    const double ih2 = g.inv_h * g.inv_h;
    const Nbr zn{z.own, z.below, z.above}, pn{p.own, p.below, p.above};
    if (first) k_pcg_matvec<true><<<grid, kPT, 0, s>>>(g, zn, pn, pout, q, sc, ih2, partials);
    else k_pcg_matvec<false><<<grid, kPT, 0, s>>>(g, zn, pn, pout, q, sc, ih2, partials);
    k_pcg_reduce<<<1, 1024, 0, s>>>(g, partials, (int)grid, 1, sc + 5, nullptr, 0);
}

void launch_pcg_update(const Geom& g, double* x, const double* p, double* r, const double* q, double* sc,
                       double* partials, cudaStream_t s) {
    const unsigned grid = pcg_grid(g);
    const int64_t n2 = (int64_t)g.n * g.n * g.nzl / 2;
    k_pcg_update<<<grid, kPT, 0, s>>>(n2, g.P > 1, reinterpret_cast<double2*>(x), reinterpret_cast<const double2*>(p),
                                      reinterpret_cast<double2*>(r), reinterpret_cast<const double2*>(q), sc,
                                      partials);
    k_pcg_reduce<<<1, 1024, 0, s>>>(g, partials, (int)grid, 1, sc + 2, nullptr, 0);
}

void launch_pcg_gradient(const Geom& g, PcgNbr x, double* E4, double* halo, double* partials, double* energies,
                         cudaStream_t s) {
    const unsigned grid = pcg_grid(g);
    k_pcg_gradient<<<grid, kPT, 0, s>>>(g, Nbr{x.own, x.below, x.above}, E4, halo, partials);
    k_pcg_reduce<<<1, 1024, 0, s>>>(g, partials, (int)grid, 3, energies, nullptr, 1);
}

void launch_pcg_unsplit(const Geom& g, const double* f, double* out, cudaStream_t s) {
    const int64_t nn = (int64_t)g.n * g.n * g.nzl;
    k_pcg_unsplit<<<(unsigned)((nn + 255) / 256), 256, 0, s>>>(g, f, out);
}

}  // namespace pic
