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
#include <cstdlib>

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
// n is a power of two: every index split is a shift and a mask (no integer division).
__device__ __forceinline__ int lg2(int v) { return __ffs(v) - 1; }
__device__ __forceinline__ PairPos pair_pos(const Geom& g, int64_t p) {
    const int ln = lg2(g.n);                 // pairs per row: n / 4 = 2^(ln - 2)
    const int64_t row = p >> (ln - 2);
    PairPos q;
    q.j = 2 * (int)(p & ((g.n >> 2) - 1));
    q.y = (int)(row & g.nmask);
    q.zl = (int)(row >> ln);
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

// 256-bit accesses (LDG/STG.E.ENL2.256): four consecutive elements of a colour row.
struct Q4 {
    double v[4];
};
__device__ __forceinline__ Q4 ld4(const double* p) {
    Q4 q;
    asm volatile("ld.global.v4.f64 {%0, %1, %2, %3}, [%4];"
                 : "=d"(q.v[0]), "=d"(q.v[1]), "=d"(q.v[2]), "=d"(q.v[3]) : "l"(p));
    return q;
}
__device__ __forceinline__ void st4(double* p, const Q4& q) {
    asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(q.v[0]), "d"(q.v[1]), "d"(q.v[2]),
                 "d"(q.v[3])
                 : "memory");
}
__device__ __forceinline__ const double* zrow(const Geom& g, const Nbr& f, int c, int zl, int y, int j) {
    const double* b = f.own;
    if (zl < 0) { b = f.below; zl += g.nzl; }
    else if (zl >= g.nzl) { b = f.above; zl -= g.nzl; }
    return b + sidx(g, c, zl, y, j);
}

// z-march work mapping of the 4-element / octet kernels: a CTA owns R = 256 / (n/8)
// consecutive rows (n/8 items per row) and walks a chunk of cz planes, so the planes
// zl -+ 1 a stencil reads were (or will be) this CTA's own rows one plane before
// (after) -- L1/L2 hits instead of DRAM re-reads (ncu: the grid-stride order re-read
// 2.7x the matvec's and 1.2x the half-sweep's algorithmic bytes).
struct ZMarch {
    int y, j, z0, z1;     // thread's row and element, the CTA's planes [z0, z1)
    bool on;
};
__device__ __forceinline__ ZMarch zmarch(const Geom& g, int cz) {
    const int qpr = g.n >> 3;                          // items per row
    const int R = min(kPT / qpr, g.n);                 // rows per CTA
    const int nyb = g.n / R;
    ZMarch m;
    const int t = threadIdx.x, rr = t / qpr;
    m.on = rr < R;
    m.j = 4 * (t - rr * qpr);
    m.y = (blockIdx.x % nyb) * R + rr;
    m.z0 = (blockIdx.x / nyb) * cz;
    m.z1 = min(m.z0 + cz, g.nzl);
    return m;
}

// The half-sweep with four elements j .. j+3 per thread (j = 0 mod 4): every row of
// the stencil is one 256-bit load, so a thread issues 8 loads for 4 updates (k_sor: 8
// for 2).  Same arithmetic and order as k_sor (bit-identical results).
template <int MODE, bool DOT>
__global__ void __launch_bounds__(kPT) k_sor4(Geom g, int c, const double* __restrict__ r, Nbr z, double* zout,
                                              double c1, double c2, double h2, int cz,
                                              double* __restrict__ partials) {
    const int hn = g.n >> 1, oc = c ^ 1;
    double acc = 0.0;
    const ZMarch zm = zmarch(g, cz);
    for (int zl = zm.z0; zm.on && zl < zm.z1; ++zl) {
        const int j = zm.j, y = zm.y;
        const int o = (y + zl + c) & 1;                          // x of element j is 2j + o
        const int64_t me = sidx(g, c, zl, y, j);
        const Q4 rv = ld4(r + me);
        Q4 zn, m;
        if (MODE == 2) {
#pragma unroll
            for (int q = 0; q < 4; ++q) zn.v[q] = __dmul_rn(c2, __dmul_rn(h2, rv.v[q]));
        } else {
            m = ld4(zrow(g, z, oc, zl, y, j));
            const double e = o ? *zrow(g, z, oc, zl, y, (j + 4) & (hn - 1)) : *zrow(g, z, oc, zl, y, (j - 1) & (hn - 1));
            const Q4 ym = ld4(zrow(g, z, oc, zl, (y - 1) & g.nmask, j));
            const Q4 yp = ld4(zrow(g, z, oc, zl, (y + 1) & g.nmask, j));
            const Q4 zm = ld4(zrow(g, z, oc, zl - 1, y, j));
            const Q4 zp = ld4(zrow(g, z, oc, zl + 1, y, j));
            Q4 zo;
            if (MODE == 0) zo = ld4(z.own + me);
            // other colour at j - 1 + o .. j + 4 + o - 1: element q has x-neighbours w[q], w[q + 1]
            const double w[5] = {o ? m.v[0] : e, o ? m.v[1] : m.v[0], o ? m.v[2] : m.v[1], o ? m.v[3] : m.v[2],
                                 o ? e : m.v[3]};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const double sq = nsum(w[q], w[q + 1], ym.v[q], yp.v[q], zm.v[q], zp.v[q]);
                const double zq = MODE == 0 ? zo.v[q] : 0.0;
                zn.v[q] = __dadd_rn(__dmul_rn(c1, zq), __dmul_rn(c2, __dadd_rn(__dmul_rn(h2, rv.v[q]), sq)));
            }
        }
        st4(zout + me, zn);
        if (DOT) {
            const Q4 ro = ld4(r + sidx(g, oc, zl, y, j));
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                acc = fma(rv.v[q], zn.v[q], acc);
                acc = fma(ro.v[q], m.v[q], acc);
            }
        }
    }
    if (DOT) block_partials(&acc, 1, partials);
    if (g.P > 1) __threadfence_system();
}

// sum_m rho_m, rho_m = dscale * raw_m (the raw CIC sums of the pitched rho planes).
__global__ void __launch_bounds__(kPT) k_pcg_rho_sum(Geom g, const double* __restrict__ raw, double dscale,
                                                     double* __restrict__ partials) {
    const int64_t npair = (int64_t)g.n * g.nzl * (g.n >> 2) * 2;   // natural pairs
    const int hq = g.n >> 1;
    double acc = 0.0;
    for (int64_t p = (int64_t)blockIdx.x * kPT + threadIdx.x; p < npair; p += (int64_t)gridDim.x * kPT) {
        const int64_t row = p >> (lg2(g.n) - 1);
        const int x = 2 * (int)(p & (hq - 1));
        const double2 v = *reinterpret_cast<const double2*>(raw + row * g.rp + x);
        acc += __dmul_rn(dscale, v.x);
        acc += __dmul_rn(dscale, v.y);
    }
    block_partials(&acc, 1, partials);
}

// ------------------------------------------------ natural octets (8 nodes) ---
// A thread takes the nodes x = 2j .. 2j+7 (j = 0 mod 4) of one row: colour elements
// j .. j+3 of both colours, one 256-bit load per colour and stencil row (12 loads for
// 8 nodes, the pair kernels above needed 12 for 2).  Node k of the octet is element
// k/2 of colour (c0 + k) & 1, c0 = (y + zl) & 1.
struct Oct {
    Q4 e, o;     // even / odd nodes of the octet
    __device__ __forceinline__ double at(int k) const { return (k & 1) ? o.v[k >> 1] : e.v[k >> 1]; }
};
__device__ __forceinline__ Oct ldoct(const Geom& g, const Nbr& f, int zl, int y, int j) {
    const int c0 = (y + zl) & 1;
    Oct r;
    r.e = ld4(zrow(g, f, c0, zl, y, j));
    r.o = ld4(zrow(g, f, c0 ^ 1, zl, y, j));
    return r;
}
__device__ __forceinline__ void stoct(const Geom& g, double* f, int zl, int y, int j, const double v[8]) {
    const int c0 = (y + zl) & 1;
    Q4 e, o;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        e.v[q] = v[2 * q];
        o.v[q] = v[2 * q + 1];
    }
    st4(f + sidx(g, c0, zl, y, j), e);
    st4(f + sidx(g, c0 ^ 1, zl, y, j), o);
}
struct Hood8 {
    Oct c, ym, yp, zm, zp;
    double left, right;      // nodes 2j - 1 and 2j + 8
};
__device__ __forceinline__ Hood8 ldhood8(const Geom& g, const Nbr& f, int zl, int y, int j) {
    const int hn = g.n >> 1, c0 = (y + zl) & 1;
    Hood8 h;
    h.c = ldoct(g, f, zl, y, j);
    h.left = *zrow(g, f, c0 ^ 1, zl, y, (j - 1) & (hn - 1));
    h.right = *zrow(g, f, c0, zl, y, (j + 4) & (hn - 1));
    h.ym = ldoct(g, f, zl, (y - 1) & g.nmask, j);
    h.yp = ldoct(g, f, zl, (y + 1) & g.nmask, j);
    h.zm = ldoct(g, f, zl - 1, y, j);
    h.zp = ldoct(g, f, zl + 1, y, j);
    return h;
}
// h <- h + beta hp, element by element (p' = z + beta p on the whole stencil)
__device__ __forceinline__ void axpy_hood8(Hood8& h, const Hood8& hp, double beta) {
    auto u4 = [&](Q4& a, const Q4& b) {
#pragma unroll
        for (int q = 0; q < 4; ++q) a.v[q] = __dadd_rn(a.v[q], __dmul_rn(beta, b.v[q]));
    };
    auto u8 = [&](Oct& a, const Oct& b) { u4(a.e, b.e); u4(a.o, b.o); };
    u8(h.c, hp.c); u8(h.ym, hp.ym); u8(h.yp, hp.yp); u8(h.zm, hp.zm); u8(h.zp, hp.zp);
    h.left = __dadd_rn(h.left, __dmul_rn(beta, hp.left));
    h.right = __dadd_rn(h.right, __dmul_rn(beta, hp.right));
}
// -Delta_h at the octet (D#26): (6 x - nb) * ih2, nb in the oracle's order.
__device__ __forceinline__ void apply_A8(const Hood8& h, double ih2, double out[8]) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const double xm = k == 0 ? h.left : h.c.at(k - 1);
        const double xp = k == 7 ? h.right : h.c.at(k + 1);
        const double sk = nsum(xm, xp, h.ym.at(k), h.yp.at(k), h.zm.at(k), h.zp.at(k));
        out[k] = __dmul_rn(__dsub_rn(__dmul_rn(6.0, h.c.at(k)), sk), ih2);
    }
}
struct OctPos {
    int zl, y, j;
    int64_t row;
};

// r = (rho - mean) - A x (D#27), partials of (b, b) and (r, r).  Thread = octet.
__global__ void __launch_bounds__(kPT) k_pcg_resid0_8(Geom g, const double* __restrict__ raw, double dscale,
                                                      const double* __restrict__ sc, double nn, Nbr x,
                                                      double* __restrict__ r, double ih2, int cz,
                                                      double* __restrict__ partials) {
    const double mean = sc[0] / nn;
    double acc[2] = {0.0, 0.0};
    const ZMarch zm = zmarch(g, cz);
    for (int zl = zm.z0; zm.on && zl < zm.z1; ++zl) {
        OctPos q;
        q.zl = zl;
        q.y = zm.y;
        q.j = zm.j;
        q.row = (int64_t)zl * g.n + zm.y;
        const double* rp = raw + q.row * g.rp + 2 * q.j;
        const Q4 v0 = ld4(rp), v1 = ld4(rp + 4);
        double ax[8], rv[8];
        apply_A8(ldhood8(g, x, q.zl, q.y, q.j), ih2, ax);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const double b = __dsub_rn(__dmul_rn(dscale, k < 4 ? v0.v[k] : v1.v[k - 4]), mean);
            rv[k] = __dsub_rn(b, ax[k]);
            acc[0] = fma(b, b, acc[0]);
            acc[1] = fma(rv[k], rv[k], acc[1]);
        }
        stoct(g, r, q.zl, q.y, q.j, rv);
    }
    block_partials(acc, 2, partials);
}

// p' = z + beta p (first: p' = z), q = A p', partial (p', q); thread = octet.
template <bool FIRST>
__global__ void __launch_bounds__(kPT) k_pcg_matvec8(Geom g, Nbr z, Nbr p, double* __restrict__ pout,
                                                     double* __restrict__ qo, const double* __restrict__ sc,
                                                     double ih2, int cz, double* __restrict__ partials) {
    const double beta = FIRST ? 0.0 : sc[3] / sc[4];
    double acc = 0.0;
    const ZMarch zm = zmarch(g, cz);
    for (int zl = zm.z0; zm.on && zl < zm.z1; ++zl) {
        OctPos q;
        q.zl = zl;
        q.y = zm.y;
        q.j = zm.j;
        q.row = (int64_t)zl * g.n + zm.y;
        Hood8 h = ldhood8(g, z, q.zl, q.y, q.j);
        if (!FIRST) axpy_hood8(h, ldhood8(g, p, q.zl, q.y, q.j), beta);
        double av[8], pv[8];
        apply_A8(h, ih2, av);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            pv[k] = h.c.at(k);
            acc = fma(pv[k], av[k], acc);
        }
        stoct(g, pout, q.zl, q.y, q.j, pv);
        stoct(g, qo, q.zl, q.y, q.j, av);
    }
    block_partials(&acc, 1, partials);
    if (g.P > 1) __threadfence_system();
}

// E = -grad_h phi (D#30) -> E4 node records (+ plane 0 into `halo`), E_d^2 partials.
__global__ void __launch_bounds__(kPT) k_pcg_gradient8(Geom g, Nbr x, double* __restrict__ E4, double* halo,
                                                       int cz, double* __restrict__ partials) {
    const double cc = 0.5 * g.inv_h;
    double e2[3] = {0.0, 0.0, 0.0};
    const ZMarch zm = zmarch(g, cz);
    for (int zl = zm.z0; zm.on && zl < zm.z1; ++zl) {
        OctPos q;
        q.zl = zl;
        q.y = zm.y;
        q.j = zm.j;
        q.row = (int64_t)zl * g.n + zm.y;
        const Hood8 h = ldhood8(g, x, q.zl, q.y, q.j);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const double xm = k == 0 ? h.left : h.c.at(k - 1);
            const double xp = k == 7 ? h.right : h.c.at(k + 1);
            const double ex = __dmul_rn(__dsub_rn(xm, xp), cc);
            const double ey = __dmul_rn(__dsub_rn(h.ym.at(k), h.yp.at(k)), cc);
            const double ez = __dmul_rn(__dsub_rn(h.zm.at(k), h.zp.at(k)), cc);
            const int64_t nd = 4 * (q.row * g.n + 2 * q.j + k);
            asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(E4 + nd), "d"(ex), "d"(ey), "d"(ez),
                         "d"(0.0) : "memory");
            if (halo && q.zl == 0)
                asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(halo + nd), "d"(ex), "d"(ey),
                             "d"(ez), "d"(0.0) : "memory");
            e2[0] = fma(ex, ex, e2[0]);
            e2[1] = fma(ey, ey, e2[1]);
            e2[2] = fma(ez, ez, e2[2]);
        }
    }
    block_partials(e2, 3, partials);
    if (halo && g.P > 1) __threadfence_system();
}

// x += alpha p ; r -= alpha q ; partial (r, r) -- 256-bit streams.
__global__ void __launch_bounds__(kPT) k_pcg_update4(int64_t n4, int sys_fence, double* __restrict__ x,
                                                     const double* __restrict__ p, double* __restrict__ r,
                                                     const double* __restrict__ q, const double* __restrict__ sc,
                                                     double* __restrict__ partials) {
    const double alpha = sc[3] / sc[5];
    double acc = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * kPT + threadIdx.x; i < n4; i += (int64_t)gridDim.x * kPT) {
        const Q4 pv = ld4(p + 4 * i), qv = ld4(q + 4 * i);
        Q4 xv = ld4(x + 4 * i), rv = ld4(r + 4 * i);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            xv.v[k] = __dadd_rn(xv.v[k], __dmul_rn(alpha, pv.v[k]));
            rv.v[k] = __dsub_rn(rv.v[k], __dmul_rn(alpha, qv.v[k]));
            acc = fma(rv.v[k], rv.v[k], acc);
        }
        st4(x + 4 * i, xv);
        st4(r + 4 * i, rv);
    }
    block_partials(&acc, 1, partials);
    if (sys_fence) __threadfence_system();     // x is read by the neighbour slabs
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


// ------------------------------------------------ temporally blocked SSOR ----
// One SSOR "pass": ns <= kTB consecutive half-sweeps (colours = bits of seq) in one
// kernel, so z and r stream through HBM once per pass instead of once per
// half-sweep (24 B/node per pass vs 16 B/node per half-sweep; 4 half-sweeps per
// pass -> 2.7x less traffic for M^-1).  Work unit = an x-y tile of tx colour
// elements x ty rows, marched along a chunk [zs, ze) of planes; the tile carries a
// halo (kHe elements, kHy rows) that shrinks by one node per half-sweep, and the
// chunk a halo of ns planes (ghost zones: the halo is recomputed redundantly, only
// the interior is written).  Planes stream through a shared-memory ring (cp.async,
// one plane ahead); at front plane f, half-sweep t updates plane f - t in place,
// which already holds half-sweep t-1's result at f - t + 1 and not yet t+1's at
// f - t - 1: the pipeline reproduces the sequential half-sweep order exactly (same
// arithmetic as k_sor, bit-identical).  Input zin and output zout are different
// buffers (neighbour tiles and ranks read zin's halo while this one writes).
constexpr int kTB = 4;                    // half-sweeps per pass
constexpr int kTX = 32;                   // interior colour elements per tile row (64 nodes)
constexpr int kTY = 8;                    // interior rows per tile
constexpr int kHe = 4;                    // x halo in elements (>= ceil(kTB/2) + 1; even: 16-B loads)
constexpr int kHy = kTB;                  // y halo in rows
constexpr int kWe = kTX + 2 * kHe;        // 40
constexpr int kWy = kTY + 2 * kHy;        // 16
constexpr int kSlots = 8;                 // ring (>= kTB + 3: ns + 2 live planes + one prefetched); slot = p & 7
constexpr int kSlot = 2 * kWy * kWe;      // doubles per slot (both colours)
constexpr int kTBThreads = 256;
// elements per thread per half-sweep: the largest region (the first half-sweep's,
// (kTY + 2 (kTB - 1)) rows x (kTX + 2 (kTB / 2)) elements) over the CTA's threads
constexpr int kMaxK = ((kTY + 2 * (kTB - 1)) * (kTX + 2 * (kTB / 2)) + kTBThreads - 1) / kTBThreads;
constexpr size_t kTBSmem = sizeof(double) * kSlots * kSlot;

__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

__global__ void __launch_bounds__(kTBThreads, 2) k_ssor_tb(Geom g, Nbr r, Nbr zin, double* __restrict__ zout,
                                                           int ns, int seq, int zero_in, int dot, int cz,
                                                           double c1, double c2, double h2,
                                                           double* __restrict__ partials) {
    static_assert((kSlots & (kSlots - 1)) == 0 && kSlots >= kTB + 3, "ring");
    static_assert(kHe % 2 == 0 && kTX % 2 == 0, "16-byte pairs");
    extern __shared__ double sm[];
    constexpr int kCP = kWy * kWe;                                    // doubles per colour plane
    constexpr int kLd = (kCP + kTBThreads - 1) / kTBThreads;          // 16-B plane loads per thread (2 colours)
    const int hn = g.n >> 1, tid = threadIdx.x;
    const int tx = min(kTX, hn), ty = min(kTY, g.n);
    const int We = tx + 2 * kHe, Wy = ty + 2 * kHy, Wp = We / 2;
    const int ntx = hn / tx, nty = g.n / ty, nzc = (g.nzl + cz - 1) / cz;
    const int nunits = ntx * nty * nzc;
    const int64_t pstride = (int64_t)g.n * hn;                        // plane stride of a colour half grid
    const int64_t cstride = (int64_t)g.nzl * pstride;                 // colour stride of a field
    const int zmask = g.nzl - 1;                                      // nzl is a power of two
    // plane p in [-nzl, 2 nzl) of field f, colour c: the slab below / this / above
    auto plane_ptr = [&](const Nbr& f, int c, int p) {
        const double* b = p < 0 ? f.below : (p > zmask ? f.above : f.own);
        return b + c * cstride + (int64_t)(p & zmask) * pstride;
    };
    double acc = 0.0;
    // element lists per half-sweep t: shared offset row * kWe + e (-1: none)
    int soff[kTB][kMaxK];
#pragma unroll
    for (int t = 0; t < kTB; ++t) {
        const int h = ns - 1 - t, a = (ns - t) / 2;
        const int nr = ty + 2 * h, ne = tx + 2 * a, r0 = kHy - h, e0 = kHe - a;
#pragma unroll
        for (int k = 0; k < kMaxK; ++k) {
            const int i = tid + k * kTBThreads;
            soff[t][k] = (t < ns && i < nr * ne) ? (r0 + i / ne) * kWe + e0 + i % ne : -1;
        }
    }
    for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
        const int bx = u % ntx, by = (u / ntx) % nty, bz = u / (ntx * nty);
        const int j0 = bx * tx - kHe, y0 = by * ty - kHy;
        const int zs = bz * cz, ze = min(zs + cz, g.nzl);
        // global in-plane offsets y * hn + j of the elements, and a bitmask of row parities
        int goff[kTB][kMaxK];
        unsigned ypar = 0;
#pragma unroll
        for (int t = 0; t < kTB; ++t)
#pragma unroll
            for (int k = 0; k < kMaxK; ++k) {
                const int so = soff[t][k] < 0 ? 0 : soff[t][k];
                const int yg = (y0 + so / kWe) & g.nmask, jg = (j0 + so % kWe) & (hn - 1);
                goff[t][k] = yg * hn + jg;
                ypar |= (unsigned)(yg & 1) << (t * kMaxK + k);
            }
        // 16-byte plane loads: pair index -> colour, row, element pair
        int lsrc[2 * kLd], ldst[2 * kLd];
#pragma unroll
        for (int k = 0; k < 2 * kLd; ++k) {
            const int i = tid + k * kTBThreads;
            const int c = i / (Wy * Wp), rem = i - c * Wy * Wp, row = rem / Wp, e = 2 * (rem - row * Wp);
            const int yg = (y0 + row) & g.nmask, jg = (j0 + e) & (hn - 1);
            lsrc[k] = i < 2 * Wy * Wp ? (c << 30) | (yg * hn + jg) : -1;
            ldst[k] = c * kCP + row * kWe + e;
        }
        // write-back pairs: one (colour, row, element pair) of the interior per thread
        const int nwb = ty * tx;                       // pairs of both colours = 2 * ty * tx / 2
        int wsm = -1, wgl = 0, wc = 0;
        if (tid < nwb) {
            const int hp = tx / 2, c = tid / (ty * hp), rem = tid - c * ty * hp, row = rem / hp, e = 2 * (rem - row * hp);
            wc = c;
            wsm = c * kCP + (kHy + row) * kWe + kHe + e;
            wgl = ((y0 + kHy + row) & g.nmask) * hn + ((j0 + kHe + e) & (hn - 1));
        }
        auto load = [&](int p) {
            double* dst = sm + (p & (kSlots - 1)) * kSlot;
            if (zero_in) {
#pragma unroll
                for (int k = 0; k < 2 * kLd; ++k)
                    if (lsrc[k] >= 0) *reinterpret_cast<double2*>(dst + ldst[k]) = make_double2(0.0, 0.0);
            } else {
                const double* b0 = plane_ptr(zin, 0, p);
                const double* b1 = plane_ptr(zin, 1, p);
#pragma unroll
                for (int k = 0; k < 2 * kLd; ++k)
                    if (lsrc[k] >= 0)
                        cp_async16(dst + ldst[k], ((lsrc[k] >> 30) ? b1 : b0) + (lsrc[k] & 0x3fffffff));
            }
            cp_async_commit();
        };
        auto load_r = [&](int f, double (&rv)[kTB][kMaxK]) {
#pragma unroll
            for (int t = 0; t < kTB; ++t) {
                const int p = f - 1 - t, h = ns - 1 - t;
                if (t < ns && p >= zs - h && p < ze + h) {
                    const double* rp = plane_ptr(r, (seq >> t) & 1, p);
#pragma unroll
                    for (int k = 0; k < kMaxK; ++k)
                        if (soff[t][k] >= 0) rv[t][k] = rp[goff[t][k]];
                }
            }
        };
        auto step = [&](int f, const double (&rv)[kTB][kMaxK], double (&rn)[kTB][kMaxK]) {
            const int f1 = ze + ns;
            if (f + 1 < f1) load(f + 1);
            else cp_async_commit();                    // keep the group count uniform
            if (f + 1 < f1) load_r(f + 1, rn);         // r of the next front plane, in flight
            cp_async_wait1();                          // plane f has landed
            __syncthreads();
#pragma unroll
            for (int t = 0; t < kTB; ++t) {
                const int p = f - 1 - t, h = ns - 1 - t;
                if (t < ns && p >= zs - h && p < ze + h) {
                    const int c = (seq >> t) & 1, oc = c ^ 1;
                    const double* so = sm + (p & (kSlots - 1)) * kSlot + oc * kCP;
                    const double* som = sm + ((p - 1) & (kSlots - 1)) * kSlot + oc * kCP;
                    const double* sop = sm + ((p + 1) & (kSlots - 1)) * kSlot + oc * kCP;
                    double* sc = sm + (p & (kSlots - 1)) * kSlot + c * kCP;
                    const unsigned pc = (unsigned)(p + c) & 1u;
#pragma unroll
                    for (int k = 0; k < kMaxK; ++k) {
                        const int off = soff[t][k];
                        if (off >= 0) {
                            const int o = (int)(((ypar >> (t * kMaxK + k)) ^ pc) & 1u);
                            const double s = nsum(so[off - 1 + o], so[off + o], so[off - kWe], so[off + kWe],
                                                  som[off], sop[off]);
                            sc[off] = __dadd_rn(__dmul_rn(c1, sc[off]),
                                                __dmul_rn(c2, __dadd_rn(__dmul_rn(h2, rv[t][k]), s)));
                        }
                    }
                }
                __syncthreads();
            }
            const int p = f - ns;                      // final: write the interior of plane p
            if (p >= zs && p < ze && wsm >= 0) {
                const double2 v = *reinterpret_cast<const double2*>(sm + (p & (kSlots - 1)) * kSlot + wsm);
                const int64_t gi = wc * cstride + (int64_t)p * pstride + wgl;
                *reinterpret_cast<double2*>(zout + gi) = v;
                if (dot) {
                    const double2 rr = *reinterpret_cast<const double2*>(r.own + gi);
                    acc = fma(rr.x, v.x, fma(rr.y, v.y, acc));
                }
            }
        };
        double ra[kTB][kMaxK], rb[kTB][kMaxK];
        const int f0 = zs - ns, f1 = ze + ns;          // planes [f0, f1) stream through the ring
        load(f0);
        load_r(f0, ra);
        int f = f0;
        for (; f + 1 < f1; f += 2) {
            step(f, ra, rb);
            step(f + 1, rb, ra);
        }
        if (f < f1) step(f, ra, rb);
        cp_async_wait0();
        __syncthreads();                               // the ring is reused by the next unit
    }
    if (dot) block_partials(&acc, 1, partials);
    if (g.P > 1) __threadfence_system();
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

// Grid of the z-march kernels: (row blocks) x (plane chunks of cz), ~2048 CTAs.
unsigned zmarch_grid(const Geom& g, int* cz) {
    const int qpr = g.n >> 3, R = std::min(kPT / qpr, g.n), nyb = g.n / R;
    int c = 1;
    while (c < g.nzl && (int64_t)nyb * (g.nzl / (2 * c)) >= 2048) c *= 2;
    *cz = c;
    return (unsigned)(nyb * ((g.nzl + c - 1) / c));
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
    int cz = 1;
    const unsigned gz = zmarch_grid(g, &cz);
    k_pcg_resid0_8<<<gz, kPT, 0, s>>>(g, raw, dscale, sc, nn, Nbr{x.own, x.below, x.above}, r, ih2, cz, partials);
    k_pcg_reduce<<<1, 1024, 0, s>>>(g, partials, (int)gz, 2, sc + 1, nullptr, 0);
    (void)grid;
}

void launch_pcg_sor(const Geom& g, int colour, int mode, bool dot, const double* r, PcgNbr z, double omega,
                    double* partials, double* sc, cudaStream_t s) {
    const unsigned grid = pcg_grid(g);
    const double h = g.L / (double)g.n;
    const double h2 = h * h, c1 = 1.0 - omega, c2 = omega / 6.0;
    const Nbr zn{z.own, z.below, z.above};
    double* zo = const_cast<double*>(z.own);
    static const bool two = [] { const char* e = getenv("PIC_PCG_SOR2"); return e && e[0] == '1'; }();
    if (two) {   // two elements per thread (the earlier kernel; A/B switch)
        if (mode == 2) k_sor<2, false><<<grid, kPT, 0, s>>>(g, colour, r, zn, zo, c1, c2, h2, partials);
        else if (mode == 1) k_sor<1, false><<<grid, kPT, 0, s>>>(g, colour, r, zn, zo, c1, c2, h2, partials);
        else if (dot) k_sor<0, true><<<grid, kPT, 0, s>>>(g, colour, r, zn, zo, c1, c2, h2, partials);
        else k_sor<0, false><<<grid, kPT, 0, s>>>(g, colour, r, zn, zo, c1, c2, h2, partials);
    } else {
        int cz = 1;
        const unsigned gz = zmarch_grid(g, &cz);
        if (mode == 2) k_sor4<2, false><<<gz, kPT, 0, s>>>(g, colour, r, zn, zo, c1, c2, h2, cz, partials);
        else if (mode == 1) k_sor4<1, false><<<gz, kPT, 0, s>>>(g, colour, r, zn, zo, c1, c2, h2, cz, partials);
        else if (dot) k_sor4<0, true><<<gz, kPT, 0, s>>>(g, colour, r, zn, zo, c1, c2, h2, cz, partials);
        else k_sor4<0, false><<<gz, kPT, 0, s>>>(g, colour, r, zn, zo, c1, c2, h2, cz, partials);
        if (dot) {
            k_pcg_reduce<<<1, 1024, 0, s>>>(g, partials, (int)gz, 1, sc + 3, sc + 4, 0);
            return;
        }
    }
    if (dot) k_pcg_reduce<<<1, 1024, 0, s>>>(g, partials, (int)grid, 1, sc + 3, sc + 4, 0);
}

int pcg_tb_stages() { return kTB; }

void launch_pcg_ssor_pass(const Geom& g, int ns, int seq, bool zero_in, bool dot, PcgNbr r, PcgNbr zin,
                          double* zout, double omega, double* partials, double* sc, cudaStream_t s) {
    static unsigned attr = 0;          // per device (bit d): the opt-in is a device attribute
    int dev = 0, sms = 148, occ = 1;
    cudaGetDevice(&dev);
    if (dev < 32 && !(attr & (1u << dev)) &&
        cudaFuncSetAttribute(k_ssor_tb, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTBSmem) == cudaSuccess)
        attr |= 1u << dev;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_ssor_tb, kTBThreads, kTBSmem);
    const int hn = g.n >> 1, tx = std::min(kTX, hn), ty = std::min(kTY, g.n);
    const int cz = std::min(g.nzl, 64);
    const int64_t units = (int64_t)(hn / tx) * (g.n / ty) * ((g.nzl + cz - 1) / cz);
    const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(units, (int64_t)std::max(occ, 1) * sms));
    const double h = g.L / (double)g.n;
    k_ssor_tb<<<grid, kTBThreads, kTBSmem, s>>>(g, Nbr{r.own, r.below, r.above}, Nbr{zin.own, zin.below, zin.above},
                                                zout, ns, seq, zero_in ? 1 : 0, dot ? 1 : 0, cz, 1.0 - omega,
                                                omega / 6.0, h * h, partials);
    if (dot) k_pcg_reduce<<<1, 1024, 0, s>>>(g, partials, (int)grid, 1, sc + 3, sc + 4, 0);
}

void launch_pcg_matvec(const Geom& g, bool first, PcgNbr z, PcgNbr p, double* pout, double* q, double* sc,
                       double* partials, cudaStream_t s) {
    const unsigned grid = pcg_grid(g);
    const double ih2 = g.inv_h * g.inv_h;
    const Nbr zn{z.own, z.below, z.above}, pn{p.own, p.below, p.above};
    int cz = 1;
    const unsigned gz = zmarch_grid(g, &cz);
    if (first) k_pcg_matvec8<true><<<gz, kPT, 0, s>>>(g, zn, pn, pout, q, sc, ih2, cz, partials);
    else k_pcg_matvec8<false><<<gz, kPT, 0, s>>>(g, zn, pn, pout, q, sc, ih2, cz, partials);
    k_pcg_reduce<<<1, 1024, 0, s>>>(g, partials, (int)gz, 1, sc + 5, nullptr, 0);
    (void)grid;
}

void launch_pcg_update(const Geom& g, double* x, const double* p, double* r, const double* q, double* sc,
                       double* partials, cudaStream_t s) {
    const unsigned grid = pcg_grid(g);
    const int64_t n4 = (int64_t)g.n * g.n * g.nzl / 4;
    k_pcg_update4<<<grid, kPT, 0, s>>>(n4, g.P > 1, x, p, r, q, sc, partials);
    k_pcg_reduce<<<1, 1024, 0, s>>>(g, partials, (int)grid, 1, sc + 2, nullptr, 0);
}

void launch_pcg_gradient(const Geom& g, PcgNbr x, double* E4, double* halo, double* partials, double* energies,
                         cudaStream_t s) {
    const unsigned grid = pcg_grid(g);
    int cz = 1;
    const unsigned gz = zmarch_grid(g, &cz);
    k_pcg_gradient8<<<gz, kPT, 0, s>>>(g, Nbr{x.own, x.below, x.above}, E4, halo, cz, partials);
    k_pcg_reduce<<<1, 1024, 0, s>>>(g, partials, (int)gz, 3, energies, nullptr, 1);
    (void)grid;
}

void launch_pcg_unsplit(const Geom& g, const double* f, double* out, cudaStream_t s) {
    const int64_t nn = (int64_t)g.n * g.n * g.nzl;
    k_pcg_unsplit<<<(unsigned)((nn + 255) / 256), 256, 0, s>>>(g, f, out);
}

}  // namespace pic
