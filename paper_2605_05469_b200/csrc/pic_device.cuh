// pic_device.cuh -- device-side helpers of the PIC hot path (sm_100a).
//
// Arithmetic that must be bit-identical between the two places it runs (the
// push-key pass and the reorder-push-deposit pass recompute the same push) is
// written once here with explicit round-to-nearest intrinsics, so no
// contraction choice of the compiler can change a result (D#17).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace pic {

// Grid geometry and step constants, passed by value to every kernel.
struct Geom {
    int n;          // cells per dimension (power of two)
    int nmask;      // n - 1
    int px;         // complex pitch of a spectral row: round_up(n/2 + 1, 8)
    int rp;         // real pitch of a grid row in doubles: 2 * px
    double L;       // domain length
    double inv_h;   // (double)n / L  (D#5)
    double dt;      // time step
    double qm_dt;   // (q/m) dt = -dt
    // Domain decomposition over P = Py Pz ranks (P = 1: the whole box), rank = pz Py + py:
    // this rank owns the cells/nodes with z in [z0, z0 + nzl), nzl = n / Pz = 2^mz, and y
    // in [y0, y0 + nyl), nyl = n / Py = 2^my (Py = 1: z-slabs, y0 = 0, nyl = n).  Local
    // real-space grids carry one extra plane (nzl) -- the ghost of the charge, the halo of
    // the field -- and, for pencils (Py > 1), one extra row per plane (nyl): nyr rows per
    // plane, n for slabs, nyl + 1 for pencils.
    int P, rank, z0, nzl, mz;
    int Py, y0, nyl, my, nyr;
    int64_t cap;    // particle capacity of this rank's arrays (sorted positions beyond it: overflow)
    // uniform external fields (Eq. 1, D#32): eext -> E += ee; boris -> Boris kick with
    // hq = (q/m) dt / 2, bt = hq B_ext, bs = 2 bt / (1 + |bt|^2)
    int eext, boris;
    double ee[3], bt[3], bs[3], hq;
};

// Index of node (ix, local row iyl, local plane izl) in a pitched real grid [nzl + 1][nyr][rp].
__device__ __forceinline__ int64_t gidx(const Geom& g, int ix, int iyl, int izl) {
    return ((int64_t)izl * g.nyr + iyl) * g.rp + ix;
}

// Local row of the node row v = (local cell row) + (0 or 1): slabs hold every row, so it
// wraps periodically; pencils hold rows 0 .. nyl (row nyl: the ghost / halo row).
__device__ __forceinline__ int yrow(const Geom& g, int v) { return g.Py > 1 ? v : (v & g.nmask); }

// Owner rank of global cell (iy, iz), and whether this rank owns it.
__device__ __forceinline__ int owner_of(const Geom& g, int iy, int iz) { return (iz >> g.mz) * g.Py + (iy >> g.my); }
__device__ __forceinline__ bool in_domain(const Geom& g, int iy, int iz) {
    return iz >= g.z0 && iz < g.z0 + g.nzl && iy >= g.y0 && iy < g.y0 + g.nyl;
}

// Cell index along one dimension: floor(x * inv_h), clamped to [0, n-1] (D#5).
__device__ __forceinline__ int cell_of(double s, int n) {
    int i = (int)floor(s);
    i = i > n - 1 ? n - 1 : i;
    return i < 0 ? 0 : i;
}

// Morton key (x fastest) of cell (ix, iy, iz), n <= 1024 (D#14).
__device__ __forceinline__ uint32_t spread3(uint32_t v) {
    v &= 0x3ffu;
    v = (v | (v << 16)) & 0x030000FFu;
    v = (v | (v << 8)) & 0x0300F00Fu;
    v = (v | (v << 4)) & 0x030C30C3u;
    v = (v | (v << 2)) & 0x09249249u;
    return v;
}
__device__ __forceinline__ uint32_t compact3(uint32_t v) {
    v &= 0x09249249u;
    v = (v ^ (v >> 2)) & 0x030C30C3u;
    v = (v ^ (v >> 4)) & 0x0300F00Fu;
    v = (v ^ (v >> 8)) & 0x030000FFu;
    v = (v ^ (v >> 16)) & 0x000003FFu;
    return v;
}
__device__ __forceinline__ uint32_t morton(int ix, int iy, int iz) {
    return spread3(ix) | (spread3(iy) << 1) | (spread3(iz) << 2);
}
__device__ __forceinline__ void unmorton(uint32_t k, int& ix, int& iy, int& iz) {
    ix = (int)compact3(k);
    iy = (int)compact3(k >> 1);
    iz = (int)compact3(k >> 2);
}

// Periodic wrap into [0, L).
__device__ __forceinline__ double wrap(double x, double L) {
    if (x >= L) {
        x = __dsub_rn(x, L);
    } else if (x < 0.0) {
        x = __dadd_rn(x, L);
        if (x >= L) x = 0.0;
    }
    return x;
}

// Global Morton key of the cell of x (the sort key of the paper-level order, D#14).
__device__ __forceinline__ uint32_t gkey_of(const Geom& g, const double x[3]) {
    int i0 = cell_of(__dmul_rn(x[0], g.inv_h), g.n);
    int i1 = cell_of(__dmul_rn(x[1], g.inv_h), g.n);
    int i2 = cell_of(__dmul_rn(x[2], g.inv_h), g.n);
    return morton(i0, i1, i2);
}

// Rank-local key of cell (ix, iyl, izl) of this rank's domain: the global Morton key with
// the domain's constant bits (y bits >= my, z bits >= mz) squeezed out -- for bit
// b < m1 = min(my, mz) the triple (x, y, z), for m1 <= b < m2 = max(my, mz) the pair (x, y)
// or (x, z), above m2 x alone.  Dense on [0, n nyl nzl) and monotone with the global key on
// the domain, so the rank's sorted array is the global sorted array restricted to it; the
// low 8 bits are still x0 y0 z0 x1 y1 z1 x2 y2 (nyl >= 8, nzl >= 4), so a 256-key brick is
// 8 x 8 x 4 cells.  P = 1: the global Morton key.
__device__ __forceinline__ uint32_t spread2(uint32_t v) {
    v &= 0x3ffu;
    v = (v | (v << 8)) & 0x00FF00FFu;
    v = (v | (v << 4)) & 0x0F0F0F0Fu;
    v = (v | (v << 2)) & 0x33333333u;
    v = (v | (v << 1)) & 0x55555555u;
    return v;
}
__device__ __forceinline__ uint32_t compact2(uint32_t v) {
    v &= 0x55555555u;
    v = (v ^ (v >> 1)) & 0x33333333u;
    v = (v ^ (v >> 2)) & 0x0F0F0F0Fu;
    v = (v ^ (v >> 4)) & 0x00FF00FFu;
    v = (v ^ (v >> 8)) & 0x0000FFFFu;
    return v;
}
__device__ __forceinline__ uint32_t lkey(const Geom& g, int ix, int iyl, int izl) {
    const int m1 = g.my < g.mz ? g.my : g.mz, m2 = g.my < g.mz ? g.mz : g.my;
    const uint32_t k1 = (1u << m1) - 1u;
    const uint32_t lo = morton(ix & k1, iyl & k1, izl & k1);
    const uint32_t other = (uint32_t)(g.my > g.mz ? iyl : izl) >> m1;   // the longer local dimension
    const uint32_t mid = spread2(((uint32_t)ix >> m1) & ((1u << (m2 - m1)) - 1u)) | (spread2(other) << 1);
    return lo | (mid << (3 * m1)) | (((uint32_t)ix >> m2) << (3 * m1 + 2 * (m2 - m1)));
}
__device__ __forceinline__ void unlkey(const Geom& g, uint32_t k, int& ix, int& iyl, int& izl) {
    const int m1 = g.my < g.mz ? g.my : g.mz, m2 = g.my < g.mz ? g.mz : g.my;
    const uint32_t lo = k & ((1u << (3 * m1)) - 1u);
    const uint32_t mid = (k >> (3 * m1)) & ((1u << (2 * (m2 - m1))) - 1u);
    const uint32_t hi = k >> (3 * m1 + 2 * (m2 - m1));
    ix = (int)(compact3(lo) | (compact2(mid) << m1) | (hi << m2));
    const int other = (int)(compact2(mid >> 1) << m1);
    iyl = (int)compact3(lo >> 1) | (g.my > g.mz ? other : 0);
    izl = (int)compact3(lo >> 2) | (g.mz > g.my ? other : 0);
}

// Local key of the cell of x on this rank; *ixg / *iyg / *izg = its global cell indices.
__device__ __forceinline__ uint32_t key_of(const Geom& g, const double x[3], int* izg = nullptr,
                                           int* iyg = nullptr, int* ixg = nullptr) {
    int i0 = cell_of(__dmul_rn(x[0], g.inv_h), g.n);
    int i1 = cell_of(__dmul_rn(x[1], g.inv_h), g.n);
    int i2 = cell_of(__dmul_rn(x[2], g.inv_h), g.n);
    if (izg) *izg = i2;
    if (iyg) *iyg = i1;
    if (ixg) *ixg = i0;
    return lkey(g, i0, i1 - g.y0, i2 - g.z0);
}

// CIC weights of one position: cell index i[d] and w[d][0] = 1 - f, w[d][1] = f,
// f = x inv_h - i.
__device__ __forceinline__ void cic_weights(const Geom& g, const double x[3], int i[3],
                                            double w[3][2]) {
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        double s = __dmul_rn(x[d], g.inv_h);
        i[d] = cell_of(s, g.n);
        double f = __dsub_rn(s, (double)i[d]);
        w[d][0] = __dsub_rn(1.0, f);
        w[d][1] = f;
    }
}

// One 32-byte node record (E_x, E_y, E_z, 0) of the field grid E4[nzl + 1][nyr][n][4]:
// a single 256-bit read-only load (LDG.E.ENL2.256).
__device__ __forceinline__ void ldg_node(const double* __restrict__ p, double& ex, double& ey,
                                         double& ez) {
    double pad;
    asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
        : "=d"(ex), "=d"(ey), "=d"(ez), "=d"(pad)
        : "l"(p));
    (void)pad;
}

// CIC gather of E at x (corner order z outer, y, x inner; fma accumulation
// from 0: S:141-149, D#17).  E4 = the slab's node records (E_x, E_y, E_z, 0),
// planes 0 .. nzl (the last one the halo copy of the next slab's plane 0).
__device__ __forceinline__ void gather_E(const Geom& g, const double* __restrict__ E4,
                                         const double x[3], double ep[3]) {
    int i[3];
    double w[3][2];
    cic_weights(g, x, i, w);
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
#pragma unroll
    for (int c = 0; c < 2; ++c) {
#pragma unroll
        for (int b = 0; b < 2; ++b) {
            const int64_t row = ((int64_t)(i[2] - g.z0 + c) * g.nyr + yrow(g, i[1] - g.y0 + b)) * g.n;
#pragma unroll
            for (int a = 0; a < 2; ++a) {
                const double wt = __dmul_rn(__dmul_rn(w[0][a], w[1][b]), w[2][c]);
                const int64_t m = row + ((i[0] + a) & g.nmask);
                double ex, ey, ez;
                ldg_node(E4 + 4 * m, ex, ey, ez);
                a0 = __fma_rn(wt, ex, a0);
                a1 = __fma_rn(wt, ey, a1);
                a2 = __fma_rn(wt, ez, a2);
            }
        }
    }
    ep[0] = a0;
    ep[1] = a1;
    ep[2] = a2;
}

// Drift + wrap: x <- wrap(fma(v, dt, x)).  Shared by the
// push (which kicks first) and the reorder pass (which re-drifts from the kicked
// velocity the push stored), so both produce bit-identical x'.
__device__ __forceinline__ void drift(const Geom& g, double x[3], const double v[3]) {
#pragma unroll
    for (int d = 0; d < 3; ++d) x[d] = wrap(__fma_rn(v[d], g.dt, x[d]), g.L);
}

// The kick of the push (D#32): E += E_ext (when nonzero); B_ext = 0:
// v <- fma(qm_dt, E, v); else Boris: v- = v + hq E, v' = v- + v- x t,
// v+ = v- + v' x s, v <- v+ + hq E -- the oracle's operation order (fma where it writes fma).
__device__ __forceinline__ void kick(const Geom& g, double e[3], double v[3]) {
    if (g.eext) {
#pragma unroll
        for (int d = 0; d < 3; ++d) e[d] = __dadd_rn(e[d], g.ee[d]);
    }
    if (!g.boris) {
#pragma unroll
        for (int d = 0; d < 3; ++d) v[d] = __fma_rn(g.qm_dt, e[d], v[d]);
        return;
    }
    double vm[3], vp[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) vm[d] = __fma_rn(g.hq, e[d], v[d]);
    vp[0] = __dadd_rn(vm[0], __dsub_rn(__dmul_rn(vm[1], g.bt[2]), __dmul_rn(vm[2], g.bt[1])));
    vp[1] = __dadd_rn(vm[1], __dsub_rn(__dmul_rn(vm[2], g.bt[0]), __dmul_rn(vm[0], g.bt[2])));
    vp[2] = __dadd_rn(vm[2], __dsub_rn(__dmul_rn(vm[0], g.bt[1]), __dmul_rn(vm[1], g.bt[0])));
    const double s0 = __dadd_rn(vm[0], __dsub_rn(__dmul_rn(vp[1], g.bs[2]), __dmul_rn(vp[2], g.bs[1])));
    const double s1 = __dadd_rn(vm[1], __dsub_rn(__dmul_rn(vp[2], g.bs[0]), __dmul_rn(vp[0], g.bs[2])));
    const double s2 = __dadd_rn(vm[2], __dsub_rn(__dmul_rn(vp[0], g.bs[1]), __dmul_rn(vp[1], g.bs[0])));
    v[0] = __fma_rn(g.hq, e[0], s0);
    v[1] = __fma_rn(g.hq, e[1], s1);
    v[2] = __fma_rn(g.hq, e[2], s2);
}

// Gather + leapfrog kick-drift + wrap:
//   v <- fma(qm_dt, E_p, v) ; x <- wrap(fma(v, dt, x)).
__device__ __forceinline__ void gather_push(const Geom& g, const double* __restrict__ E4,
                                            double x[3], double v[3]) {
    double ep[3];
    gather_E(g, E4, x, ep);
    kick(g, ep, v);
    drift(g, x, v);
}

// ------------------------------------------------------- particle layout ----
// Two streams per particle i: XY[i] = (x, y) (16 B) and ZV[i] = (z, v_z, v_x, v_y)
// (32 B, one sector; as double2: ZV2[2i] = (z, v_z), ZV2[2i+1] = (v_x, v_y)).  A
// scattered gather of one particle touches 2 sectors and uses 48 of their 64 bytes
// (three 16-B streams: 3 sectors, 48 of 96); the kick rewrites exactly the ZV record.
struct PState {
    double2* xy;    // [cap]
    double2* zv;    // [2 cap]
};

__device__ __forceinline__ void ld_zv(const double2* p, double2& b, double2& c) {
    asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(b.x), "=d"(b.y), "=d"(c.x), "=d"(c.y) : "l"(p));
}
__device__ __forceinline__ void st_zv(double2* p, double2 b, double2 c) {
    asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(b.x), "d"(b.y), "d"(c.x), "d"(c.y)
                 : "memory");
}
__device__ __forceinline__ void st_zv_cs(double2* p, double2 b, double2 c) {   // streaming (evict first)
    asm volatile("st.global.cs.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(b.x), "d"(b.y), "d"(c.x), "d"(c.y)
                 : "memory");
}

__device__ __forceinline__ void load_particle(const PState& s, int64_t i, double x[3], double v[3]) {
    const double2 a = __ldg(s.xy + i);
    double2 b, c;
    ld_zv(s.zv + 2 * i, b, c);
    x[0] = a.x; x[1] = a.y; x[2] = b.x;
    v[0] = c.x; v[1] = c.y; v[2] = b.y;
}

__device__ __forceinline__ void store_particle(const PState& s, int64_t i, const double x[3],
                                               const double v[3]) {
    s.xy[i] = make_double2(x[0], x[1]);
    st_zv(s.zv + 2 * i, make_double2(x[2], v[2]), make_double2(v[0], v[1]));
}

// -------------------------------------------------------------- cp.async ----
// 16-byte global -> shared copies (LDGSTS, L2 only) and their commit groups.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
// Bulk prefetch of a contiguous global range into L2 (TMA unit; 16-B aligned, size a
// multiple of 16), issued by one thread, no completion to wait for.
__device__ __forceinline__ void prefetch_l2_bulk(const void* gmem, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(gmem), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait0() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}

// ---------------------------------------------------------------- Philox ----
// Philox4x32-10 (D#10): counter (j lo, j hi, b, 0), key (seed lo, seed hi).
__device__ __forceinline__ void philox4x32_10(uint32_t c[4], uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t lo0 = 0xD2511F53u * c[0], hi0 = __umulhi(0xD2511F53u, c[0]);
        const uint32_t lo1 = 0xCD9E8D57u * c[2], hi1 = __umulhi(0xCD9E8D57u, c[2]);
        const uint32_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
        c[0] = n0; c[1] = lo1; c[2] = n2; c[3] = lo0;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
}

}  // namespace pic
