// particle_kernels.cu -- particle side of the PIC step on sm_100a.
//
// Particle state lives in HBM as three streams of 128-bit pairs (pic_device.cuh):
// (x, y), (z, v_z), (v_x, v_y).  One step (after the solve) is four kernels:
//   push_key : stream the sorted particles, gather E (eight 256-bit node loads),
//              kick v in place, drift to x' (not stored), key of the new cell,
//              rank = count[key]++ (arrival order).
//   scan     : offs = exclusive scan of count (3 kernels, 4096-cell tiles).
//   place    : perm[offs[key] + rank] = i (no atomics).
//   reorder_deposit : one CTA per Morton brick of 256 cells (8 x 8 x 4): stable
//              order inside each cell (D#14), gather x, v' through perm, the
//              identical drift x' = wrap(x + v' dt), x', v' streamed to the stable
//              slot, CIC charge summed per cell in registers, folded into a node
//              tile in shared memory, one fp64 global reduction per node.
// The drift is computed twice from bit-identical code (pic_device.cuh) instead of
// storing x' in push_key (24 B/particle less traffic), and reorder_deposit does
// no field gather at the scattered pre-sort positions.
#include <algorithm>
#include <cstdlib>

#include "kernels.h"

namespace pic {

namespace {

constexpr int kThreads = 256;
constexpr int kBrick = 256;     // cells per reorder/deposit CTA (Morton 8 bits)
constexpr int kCap = 2048;      // particles staged per chunk (29 B of shared memory each)
constexpr int kBatch = 2;       // particles per thread with loads in flight together
__constant__ int g_dbg_mode = 0;   // experiment switch (0 = the method)

// ---------------------------------------------------------------- init -----
// Landau initial condition: x_d by Newton on the inverse CDF of
// (1 + alpha cos(k x))/L from x = u_d L (|dx| < 1e-12 or 32 iterations),
// velocities by Box-Muller from u_3..u_6, Philox counter = particle index (D#10).
__global__ void __launch_bounds__(kThreads) k_sample(Geom g, PState st, int64_t np, double k,
                                                     double alpha, uint32_t s0, uint32_t s1) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= np) return;
    double u[8];
#pragma unroll
    for (int b = 0; b < 4; ++b) {
        uint32_t c[4] = {(uint32_t)j, (uint32_t)((uint64_t)j >> 32), (uint32_t)b, 0u};
        philox4x32_10(c, s0, s1);
        const uint64_t w0 = (uint64_t)c[0] | ((uint64_t)c[1] << 32);
        const uint64_t w1 = (uint64_t)c[2] | ((uint64_t)c[3] << 32);
        u[2 * b] = (double)(w0 >> 11) * 0x1p-53;
        u[2 * b + 1] = (double)(w1 >> 11) * 0x1p-53;
    }
    const double ak = alpha / k;
    double x[3], v[3];
    for (int d = 0; d < 3; ++d) {
        const double target = u[d] * g.L;
        double xx = target;
        for (int it = 0; it < 32; ++it) {
            const double F = __dsub_rn(__dadd_rn(xx, __dmul_rn(ak, sin(k * xx))), target);
            const double dF = __dadd_rn(1.0, __dmul_rn(alpha, cos(k * xx)));
            const double dx = __ddiv_rn(F, dF);
            xx = __dsub_rn(xx, dx);
            if (fabs(dx) < 1e-12) break;
        }
        x[d] = wrap(xx, g.L);
    }
    const double two_pi = 6.283185307179586476925286766559;
    const double r1 = sqrt(-2.0 * log(1.0 - u[3]));
    const double r2 = sqrt(-2.0 * log(1.0 - u[5]));
    v[0] = r1 * cos(two_pi * u[4]);
    v[1] = r1 * sin(two_pi * u[4]);
    v[2] = r2 * cos(two_pi * u[6]);
    store_particle(st, j, x, v);
}

__global__ void __launch_bounds__(kThreads) k_soa_to_pairs(const double* __restrict__ soa, int64_t np,
                                                           PState dst) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= np) return;
    double x[3], v[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) { x[d] = soa[d * np + i]; v[d] = soa[(3 + d) * np + i]; }
    store_particle(dst, i, x, v);
}

__global__ void __launch_bounds__(kThreads) k_pairs_to_soa(PState src, int64_t np,
                                                           double* __restrict__ soa) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= np) return;
    double x[3], v[3];
    load_particle(src, i, x, v);
#pragma unroll
    for (int d = 0; d < 3; ++d) { soa[d * np + i] = x[d]; soa[(3 + d) * np + i] = v[d]; }
}

// ----------------------------------------------------------- push + key ----
// Grid-stride over the sorted particles with the next particle's loads in flight
// while the current one gathers E.  rank[i] = arrival order in the new cell
// (return value of the count atomic), so the placement needs no second atomic.
template <bool PUSH>
__global__ void __launch_bounds__(kThreads) k_push_key(Geom g, PState cur, int64_t np,
                                                       const double* __restrict__ E4,
                                                       uint32_t* __restrict__ key,
                                                       uint16_t* __restrict__ rank,
                                                       uint32_t* __restrict__ count,
                                                       int* __restrict__ err) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < np; i += stride) {
        double x[3], v[3];
        load_particle(cur, i, x, v);
        if (PUSH) {
            const double z0 = x[2];
            gather_push(g, E4, x, v);
            cur.p[1][i] = make_double2(z0, v[2]);
            cur.p[2][i] = make_double2(v[0], v[1]);
        } else if (!(x[0] >= 0.0 && x[0] < g.L && x[1] >= 0.0 && x[1] < g.L && x[2] >= 0.0 && x[2] < g.L)) {
            atomicExch(err + 1, 1);   // imported position outside [0, L)
        }
        const uint32_t k = key_of(g, x);
        key[i] = k;
        const uint32_t r = atomicAdd(count + k, 1u);
        if (r > 0xffffu) atomicExch(err, 1);
        rank[i] = (uint16_t)r;
    }
}

// The step's push: one CTA per Morton brick of 256 cells.  The particles of the
// brick are the contiguous sorted range [offs[c0], offs[c0 + 256)) and all their
// CIC corners lie in the brick's 9 x 9 x 5 node tile, which is staged in shared
// memory (13 KB of node records) with coalesced loads; the gather then reads
// shared memory.  Kick v in place, drift to x' (not stored), key, rank.
__global__ void __launch_bounds__(kThreads) k_push_key_brick(Geom g, PState cur,
                                                             const uint32_t* __restrict__ offs,
                                                             const double* __restrict__ E4,
                                                             uint32_t* __restrict__ key,
                                                             uint16_t* __restrict__ rank,
                                                             uint32_t* __restrict__ count,
                                                             int* __restrict__ err) {
    __shared__ double4 etile[9 * 9 * 5];
    const int t = threadIdx.x;
    const uint32_t c0 = blockIdx.x * kBrick;
    int bx, by, bz;
    unmorton(c0, bx, by, bz);
    for (int q = t; q < 9 * 9 * 5; q += kThreads) {
        const int nx = q % 9, ny = (q / 9) % 9, nz = q / 81;
        const int64_t m = ((int64_t)((bz + nz) & g.nmask) * g.n + ((by + ny) & g.nmask)) * g.n + ((bx + nx) & g.nmask);
        double ex, ey, ez;
        ldg_node(E4 + 4 * m, ex, ey, ez);
        etile[q] = make_double4(ex, ey, ez, 0.0);
    }
    const uint32_t P0 = __ldg(offs + c0), P1 = __ldg(offs + c0 + kBrick);
    __syncthreads();
    double xn[3], vn[3];
    if (P0 + t < P1) load_particle(cur, P0 + t, xn, vn);
    for (uint32_t i = P0 + t; i < P1; i += kThreads) {
        double x[3] = {xn[0], xn[1], xn[2]}, v[3] = {vn[0], vn[1], vn[2]};
        // next particle's loads in flight while this one waits on its count atomic
        if (i + kThreads < P1) load_particle(cur, i + kThreads, xn, vn);
        const double z0 = x[2];
        // CIC gather from the tile: same weights, corner order and fma chain as gather_E
        int ii[3];
        double w[3][2];
        cic_weights(g, x, ii, w);
        const int lx = ii[0] - bx, ly = ii[1] - by, lz = ii[2] - bz;
        double e0 = 0.0, e1 = 0.0, e2 = 0.0;
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
            for (int b = 0; b < 2; ++b)
#pragma unroll
                for (int a = 0; a < 2; ++a) {
                    const double wt = __dmul_rn(__dmul_rn(w[0][a], w[1][b]), w[2][c]);
                    const double4 e = etile[((lz + c) * 9 + (ly + b)) * 9 + (lx + a)];
                    e0 = __fma_rn(wt, e.x, e0);
                    e1 = __fma_rn(wt, e.y, e1);
                    e2 = __fma_rn(wt, e.z, e2);
                }
        v[0] = __fma_rn(g.qm_dt, e0, v[0]);
        v[1] = __fma_rn(g.qm_dt, e1, v[1]);
        v[2] = __fma_rn(g.qm_dt, e2, v[2]);
        drift(g, x, v);
        cur.p[1][i] = make_double2(z0, v[2]);    // kicked velocity in place: (x_n, v_{n+1/2})
        cur.p[2][i] = make_double2(v[0], v[1]);
        const uint32_t k = key_of(g, x);
        key[i] = k;
        const uint32_t r = atomicAdd(count + k, 1u);
        if (r > 0xffffu) atomicExch(err, 1);
        rank[i] = (uint16_t)r;
    }
}

__global__ void __launch_bounds__(kThreads) k_keys_only(Geom g, PState cur, int64_t np,
                                                        uint32_t* __restrict__ key) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= np) return;
    double x[3], v[3];
    load_particle(cur, i, x, v);
    key[i] = key_of(g, x);
}

// ------------------------------------------------------------------ scan ---
constexpr int kScanTile = kThreads * 16;   // 4096 cells per CTA

__global__ void __launch_bounds__(kThreads) k_scan_reduce(const uint32_t* __restrict__ count,
                                                          int64_t ncell, uint32_t* __restrict__ bsum) {
    __shared__ uint32_t red[kThreads / 32];
    const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * 16;
    uint32_t s = 0;
    if (base + 16 <= ncell) {
        const uint4* p = reinterpret_cast<const uint4*>(count + base);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const uint4 v = __ldg(p + q);
            s += v.x + v.y + v.z + v.w;
        }
    } else {
        for (int64_t c = base; c < ncell && c < base + 16; ++c) s += count[c];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t t = 0;
        for (int w = 0; w < kThreads / 32; ++w) t += red[w];
        bsum[blockIdx.x] = t;
    }
}

// exclusive scan of bsum[0..nb) in place by one CTA of 1024 threads
__global__ void __launch_bounds__(1024) k_scan_bsum(uint32_t* __restrict__ bsum, int nb) {
    __shared__ uint32_t ws[32];
    const int per = (nb + blockDim.x - 1) / blockDim.x;
    const int lo = threadIdx.x * per, hi = min(nb, lo + per);
    uint32_t s = 0;
    for (int i = lo; i < hi; ++i) s += bsum[i];
    // block exclusive scan of s
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t inc = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
    }
    if (lane == 31) ws[wid] = inc;
    __syncthreads();
    if (wid == 0) {
        uint32_t w = lane < (int)(blockDim.x >> 5) ? ws[lane] : 0u;
        uint32_t wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += t;
        }
        ws[lane] = wi - w;
    }
    __syncthreads();
    uint32_t run = ws[wid] + inc - s;
    for (int i = lo; i < hi; ++i) {
        const uint32_t v = bsum[i];
        bsum[i] = run;
        run += v;
    }
}

__global__ void __launch_bounds__(kThreads) k_scan_apply(const uint32_t* __restrict__ count,
                                                         uint32_t* __restrict__ offs, int64_t ncell,
                                                         const uint32_t* __restrict__ bsum) {
    __shared__ uint32_t ws[kThreads / 32];
    const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * 16;
    uint32_t v[16];
    const bool full = base + 16 <= ncell;
    if (full) {
        const uint4* p = reinterpret_cast<const uint4*>(count + base);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const uint4 t = __ldg(p + q);
            v[4 * q] = t.x; v[4 * q + 1] = t.y; v[4 * q + 2] = t.z; v[4 * q + 3] = t.w;
        }
    } else {
#pragma unroll
        for (int q = 0; q < 16; ++q) v[q] = base + q < ncell ? count[base + q] : 0u;
    }
    uint32_t s = 0;
#pragma unroll
    for (int q = 0; q < 16; ++q) s += v[q];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t inc = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
    }
    if (lane == 31) ws[wid] = inc;
    __syncthreads();
    uint32_t wpre = 0;
    for (int w = 0; w < wid; ++w) wpre += ws[w];
    uint32_t run = bsum[blockIdx.x] + wpre + inc - s;
#pragma unroll
    for (int q = 0; q < 16; ++q) {
        const uint32_t c = v[q];
        v[q] = run;
        run += c;
    }
    if (full) {
        uint4* po = reinterpret_cast<uint4*>(offs + base);
#pragma unroll
        for (int q = 0; q < 4; ++q) po[q] = make_uint4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    } else {
        for (int q = 0; q < 16; ++q)
            if (base + q < ncell) offs[base + q] = v[q];
    }
    if (ncell > base && ncell <= base + 16) offs[ncell] = run;   // owner of the last cell: total
}

// ----------------------------------------------------------------- place ---
// perm[offs[key[i]] + rank[i]] = i  (no atomics: ranks came from push_key)
__global__ void __launch_bounds__(kThreads) k_place(const uint32_t* __restrict__ key,
                                                    const uint16_t* __restrict__ rank, int64_t np,
                                                    const uint32_t* __restrict__ offs,
                                                    uint32_t* __restrict__ perm) {
    // 4 particles per thread: 16-byte key and 8-byte rank loads, 4 offset lookups in flight
    const int64_t i0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
    if (i0 >= np) return;
    if (i0 + 4 <= np) {
        const uint4 k4 = __ldg(reinterpret_cast<const uint4*>(key + i0));
        const uint2 r4 = __ldg(reinterpret_cast<const uint2*>(rank + i0));
        const uint32_t o0 = __ldg(offs + k4.x), o1 = __ldg(offs + k4.y);
        const uint32_t o2 = __ldg(offs + k4.z), o3 = __ldg(offs + k4.w);
        perm[o0 + (r4.x & 0xffffu)] = (uint32_t)i0;
        perm[o1 + (r4.x >> 16)] = (uint32_t)(i0 + 1);
        perm[o2 + (r4.y & 0xffffu)] = (uint32_t)(i0 + 2);
        perm[o3 + (r4.y >> 16)] = (uint32_t)(i0 + 3);
    } else {
        for (int64_t i = i0; i < np; ++i) perm[__ldg(offs + __ldg(key + i)) + __ldg(rank + i)] = (uint32_t)i;
    }
}

// ------------------------------------------------- reorder + push + deposit -
// Per chunk of the brick's sorted positions (whole cells, <= kCap particles):
//   A  stage perm[chunk] (coalesced); each cell's thread tags its positions with
//      the local cell id;
//   B  thread per position p: stable rank r of its particle inside the cell
//      (#perm entries of the cell below its own, broadcast reads), gather x, v'
//      through perm, re-drift, store x', v' at the stable slot s0 + r, and keep
//      the fractional offsets f = x' inv_h - i of the new position in shared
//      memory at that slot;
//   C  thread per cell: sum the 8 corner weights (w_x w_y) w_z of its particles in
//      stable order in registers.
// After the last chunk the 256 cells' sums are folded into the 9 x 9 x 5 node
// tile (eight conflict-free passes) and flushed with one fp64 RED.ADD per node.
// No atomics and no shuffles inside the CTA: the per-brick charge is deterministic.
// FRAC_SMEM: keep the fractional offsets of the new positions in shared memory
// (24 B per staged particle) for the per-cell sums; otherwise re-read x' from L2.
// v3: the gather runs as cp.async (LDGSTS, 16 B, L2 only) straight into the stable
// sorted slot of a shared-memory copy of the chunk: every thread keeps all of its
// particles' loads in flight without holding registers.  Then, with the chunk in
// shared memory in sorted order: drift in place, stream x', v' out with coalesced
// 16-byte stores, and sum the CIC weights per cell from shared memory.
constexpr int kCapA = 2048;     // particles per chunk of the cp.async variant (96 KB staged)

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}

template <bool PUSH>
__global__ void __launch_bounds__(kThreads, 2) k_reorder_deposit_async(
    Geom g, const uint32_t* __restrict__ offs, const uint32_t* __restrict__ perm, PState cur,
    PState nxt, double* __restrict__ rho, int* __restrict__ err) {
    extern __shared__ double dyn_smem[];
    double2* sp0 = reinterpret_cast<double2*>(dyn_smem);          // [kCapA] (x, y)
    double2* sp1 = sp0 + kCapA;                                     // [kCapA] (z, vz)
    double2* sp2 = sp1 + kCapA;                                     // [kCapA] (vx, vy)
    double* tile = reinterpret_cast<double*>(sp2 + kCapA);         // [9*9*5]
    uint32_t* sperm = reinterpret_cast<uint32_t*>(tile + 9 * 9 * 5);   // [kCapA]
    uint32_t* soffs = sperm + kCapA;                                // [kBrick + 1]
    uint8_t* scell = reinterpret_cast<uint8_t*>(soffs + kBrick + 1);   // [kCapA]
    const int t = threadIdx.x;
    const uint32_t c0 = blockIdx.x * kBrick;
    int bx, by, bz;
    unmorton(c0, bx, by, bz);
    soffs[t] = offs[c0 + t];
    if (t == 0) soffs[kBrick] = offs[c0 + kBrick];
    for (int q = t; q < 9 * 9 * 5; q += kThreads) tile[q] = 0.0;
    __syncthreads();

    double acc[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[q] = 0.0;
    int ca = 0;
    while (ca < kBrick) {
        if (soffs[ca + 1] - soffs[ca] > (uint32_t)kCapA) {
            if (t == 0) atomicExch(err, 1);
            return;
        }
        int lo = ca + 1, hi = kBrick;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (soffs[mid] - soffs[ca] <= (uint32_t)kCapA) lo = mid; else hi = mid - 1;
        }
        const int cb = lo;
        const uint32_t P0 = soffs[ca];
        const int cnt = (int)(soffs[cb] - P0);
        for (int p = t; p < cnt; p += kThreads) sperm[p] = __ldg(perm + P0 + p);
        const bool mine = t >= ca && t < cb;
        const int s0 = mine ? (int)(soffs[t] - P0) : 0, s1 = mine ? (int)(soffs[t + 1] - P0) : 0;
        for (int p = s0; p < s1; ++p) scell[p] = (uint8_t)t;
        __syncthreads();
        // stable rank -> cp.async of the particle into its sorted slot
        for (int p = t; p < cnt; p += kThreads) {
            const int c = scell[p];
            const int q0 = (int)(soffs[c] - P0), q1 = (int)(soffs[c + 1] - P0);
            const uint32_t j = sperm[p];
            int r = 0;
            for (int q = q0; q < q1; ++q) r += sperm[q] < j;
            const int o = q0 + r;
            cp_async16(sp0 + o, cur.p[0] + j);
            cp_async16(sp1 + o, cur.p[1] + j);
            cp_async16(sp2 + o, cur.p[2] + j);
        }
        cp_async_wait_all();
        __syncthreads();
        // drift in place (v is already kicked), coalesced streaming stores
        for (int p = t; p < cnt; p += kThreads) {
            double2 a = sp0[p], b = sp1[p];
            const double2 e = sp2[p];
            if (PUSH) {
                double x[3] = {a.x, a.y, b.x};
                const double v[3] = {e.x, e.y, b.y};
                drift(g, x, v);
                a = make_double2(x[0], x[1]);
                b = make_double2(x[2], b.y);
                sp0[p] = a;
                sp1[p] = b;
            }
            const int64_t o = (int64_t)P0 + p;
            nxt.p[0][o] = a;
            nxt.p[1][o] = b;
            nxt.p[2][o] = e;
        }
        __syncthreads();
        // CIC charge: thread per cell, its particles in stable order from shared memory
        for (int p = s0; p < s1; ++p) {
            const double2 a = sp0[p], b = sp1[p];
            const double x[3] = {a.x, a.y, b.x};
            int ii[3];
            double w[3][2];
            cic_weights(g, x, ii, w);
#pragma unroll
            for (int q = 0; q < 8; ++q)
                acc[q] = __dadd_rn(acc[q], __dmul_rn(__dmul_rn(w[0][q & 1], w[1][(q >> 1) & 1]), w[2][q >> 2]));
        }
        __syncthreads();
        ca = cb;
    }
    const int lx = (int)compact3((uint32_t)t), ly = (int)compact3((uint32_t)t >> 1),
              lz = (int)compact3((uint32_t)t >> 2);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const int a = q & 1, b = (q >> 1) & 1, c = q >> 2;
        tile[((lz + c) * 9 + (ly + b)) * 9 + (lx + a)] += acc[q];
        __syncthreads();
    }
    for (int q = t; q < 9 * 9 * 5; q += kThreads) {
        const double val = tile[q];
        if (val == 0.0) continue;
        const int nx = q % 9, ny = (q / 9) % 9, nz = q / 81;
        atomicAdd(rho + gidx(g, (bx + nx) & g.nmask, (by + ny) & g.nmask, (bz + nz) & g.nmask), val);
    }
}

template <bool PUSH, bool FRAC_SMEM, int KB = kBatch>
__global__ void __launch_bounds__(kThreads, KB > 2 ? 2 : (FRAC_SMEM ? 3 : 4)) k_reorder_deposit(
    Geom g, const uint32_t* __restrict__ offs, const uint32_t* __restrict__ perm, PState cur,
    PState nxt, double* __restrict__ rho, int* __restrict__ err) {
    extern __shared__ double dyn_smem[];
    double* tile = dyn_smem;                                                         // [9*9*5]
    double(*sfrac)[kCap] = reinterpret_cast<double(*)[kCap]>(dyn_smem + 9 * 9 * 5);  // [3][kCap]
    uint32_t* sperm = reinterpret_cast<uint32_t*>(dyn_smem + 9 * 9 * 5 + (FRAC_SMEM ? 3 * kCap : 0));
    uint32_t* soffs = sperm + kCap;                                                  // [kBrick + 1]
    uint8_t* scell = reinterpret_cast<uint8_t*>(soffs + kBrick + 1);                 // [kCap]
    const int t = threadIdx.x;
    const uint32_t c0 = blockIdx.x * kBrick;
    int bx, by, bz;
    unmorton(c0, bx, by, bz);
    soffs[t] = offs[c0 + t];
    if (t == 0) soffs[kBrick] = offs[c0 + kBrick];
    for (int q = t; q < 9 * 9 * 5; q += kThreads) tile[q] = 0.0;
    __syncthreads();

    double acc[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[q] = 0.0;
    int ca = 0;
    while (ca < kBrick) {
        // chunk = cells [ca, cb), the largest run with at most kCap particles
        if (soffs[ca + 1] - soffs[ca] > (uint32_t)kCap) {
            if (t == 0) atomicExch(err, 1);
            return;
        }
        int lo = ca + 1, hi = kBrick;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (soffs[mid] - soffs[ca] <= (uint32_t)kCap) lo = mid; else hi = mid - 1;
        }
        const int cb = lo;
        const uint32_t P0 = soffs[ca];
        const int cnt = (int)(soffs[cb] - P0);
        // A
        for (int p = t; p < cnt; p += kThreads) sperm[p] = __ldg(perm + P0 + p);
        const bool mine = t >= ca && t < cb;
        const int s0 = mine ? (int)(soffs[t] - P0) : 0, s1 = mine ? (int)(soffs[t + 1] - P0) : 0;
        for (int p = s0; p < s1; ++p) scell[p] = (uint8_t)t;
        __syncthreads();
        // B, kBatch positions per thread at a time: all their gathers in flight together
        for (int pb = t; pb < cnt; pb += KB * kThreads) {
            int o[KB];
            uint32_t j[KB];
#pragma unroll
            for (int k = 0; k < KB; ++k) {
                const int p = pb + k * kThreads;
                o[k] = -1;
                if (p < cnt) {
                    const int c = scell[p];
                    const int q0 = (int)(soffs[c] - P0), q1 = (int)(soffs[c + 1] - P0);
                    j[k] = sperm[p];
                    int r = 0;
                    if (g_dbg_mode == 1) r = p - q0;
                    else for (int q = q0; q < q1; ++q) r += sperm[q] < j[k];
                    o[k] = q0 + r;
                }
            }
            double2 a[KB], b[KB], e[KB];
#pragma unroll
            for (int k = 0; k < KB; ++k)
                if (o[k] >= 0) {
                    a[k] = __ldg(cur.p[0] + j[k]);
                    b[k] = __ldg(cur.p[1] + j[k]);
                    e[k] = __ldg(cur.p[2] + j[k]);
                }
#pragma unroll
            for (int k = 0; k < KB; ++k)
                if (o[k] >= 0) {
                    double x[3] = {a[k].x, a[k].y, b[k].x}, v[3] = {e[k].x, e[k].y, b[k].y};
                    if (PUSH) drift(g, x, v);    // v is already kicked (push_key)
                    store_particle(nxt, (int64_t)P0 + o[k], x, v);
                    if (FRAC_SMEM) {
#pragma unroll
                        for (int d = 0; d < 3; ++d) {
                            const double sd = __dmul_rn(x[d], g.inv_h);
                            sfrac[d][o[k]] = __dsub_rn(sd, (double)cell_of(sd, g.n));
                        }
                    }
                }
        }
        __syncthreads();
        // C
        for (int p = s0; p < (g_dbg_mode == 1 ? s0 : s1); ++p) {
            double fx, fy, fz;
            if (FRAC_SMEM) {
                fx = sfrac[0][p]; fy = sfrac[1][p]; fz = sfrac[2][p];
            } else {   // this block's own stores, visible after the barrier; L2 reads
                const double2 xy = __ldcg(nxt.p[0] + P0 + p);
                const double2 zv = __ldcg(nxt.p[1] + P0 + p);
                const double x3[3] = {xy.x, xy.y, zv.x};
                double f3[3];
#pragma unroll
                for (int d = 0; d < 3; ++d) {
                    const double sd = __dmul_rn(x3[d], g.inv_h);
                    f3[d] = __dsub_rn(sd, (double)cell_of(sd, g.n));
                }
                fx = f3[0]; fy = f3[1]; fz = f3[2];
            }
            const double wx[2] = {__dsub_rn(1.0, fx), fx}, wy[2] = {__dsub_rn(1.0, fy), fy},
                         wz[2] = {__dsub_rn(1.0, fz), fz};
#pragma unroll
            for (int q = 0; q < 8; ++q)
                acc[q] = __dadd_rn(acc[q], __dmul_rn(__dmul_rn(wx[q & 1], wy[(q >> 1) & 1]), wz[q >> 2]));
        }
        __syncthreads();
        ca = cb;
    }
    // fold the cell sums into the node tile: pass q adds corner q of every cell
    const int lx = (int)compact3((uint32_t)t), ly = (int)compact3((uint32_t)t >> 1),
              lz = (int)compact3((uint32_t)t >> 2);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const int a = q & 1, b = (q >> 1) & 1, c = q >> 2;
        tile[((lz + c) * 9 + (ly + b)) * 9 + (lx + a)] += acc[q];
        __syncthreads();
    }
    for (int q = t; q < 9 * 9 * 5; q += kThreads) {
        const double val = tile[q];
        if (val == 0.0) continue;
        const int nx = q % 9, ny = (q / 9) % 9, nz = q / 81;
        atomicAdd(rho + gidx(g, (bx + nx) & g.nmask, (by + ny) & g.nmask, (bz + nz) & g.nmask), val);
    }
}

__global__ void __launch_bounds__(kThreads) k_half_kick(Geom g, PState cur, int64_t np,
                                                        const double* __restrict__ E4) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= np) return;
    double x[3], v[3], ep[3];
    load_particle(cur, i, x, v);
    gather_E(g, E4, x, ep);
    const double hk = -0.5 * g.qm_dt;   // v_{-1/2} = v_0 - (q/m) E dt/2
#pragma unroll
    for (int d = 0; d < 3; ++d) v[d] = __fma_rn(hk, ep[d], v[d]);
    store_particle(cur, i, x, v);
}

// perm segments of every cell sorted ascending in place (export of the stable
// permutation; the step itself ranks them in shared memory only).
__global__ void __launch_bounds__(kThreads) k_sort_segments(const uint32_t* __restrict__ offs,
                                                            int64_t ncell, uint32_t* __restrict__ perm) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= ncell) return;
    const uint32_t s0 = offs[c], s1 = offs[c + 1];
    for (uint32_t a = s0 + 1; a < s1; ++a) {
        const uint32_t vv = perm[a];
        uint32_t b = a;
        while (b > s0 && perm[b - 1] > vv) { perm[b] = perm[b - 1]; --b; }
        perm[b] = vv;
    }
}

inline unsigned blocks(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

constexpr size_t kReorderAsyncSmem = sizeof(double2) * 3 * kCapA + sizeof(double) * 9 * 9 * 5 +
                                      sizeof(uint32_t) * (kCapA + kBrick + 1) + kCapA;
constexpr size_t reorder_smem(bool frac) {
    return sizeof(double) * ((frac ? 3 * kCap : 0) + 9 * 9 * 5) + sizeof(uint32_t) * (kCap + kBrick + 1) + kCap;
}
int g_reorder_variant = -1;   // 1: fractional offsets staged in shared memory, 0: re-read from L2
bool reorder_frac_smem() {
    if (g_reorder_variant < 0) {
        const char* e = getenv("PIC_REORDER_FRAC_SMEM");
        g_reorder_variant = e ? atoi(e) != 0 : 1;
        const char* m = getenv("PIC_DBG_MODE");
        if (m) { int v = atoi(m); cudaMemcpyToSymbol(g_dbg_mode, &v, sizeof(int)); }
    }
    return g_reorder_variant != 0;
}

}  // namespace

void launch_sample(const Geom& g, PState st, int64_t np, double k, double alpha, uint64_t seed,
                   cudaStream_t s) {
    if (np == 0) return;
    k_sample<<<blocks(np, kThreads), kThreads, 0, s>>>(g, st, np, k, alpha, (uint32_t)seed,
                                                        (uint32_t)(seed >> 32));
}

void launch_soa_to_pairs(const double* soa, int64_t np, PState dst, cudaStream_t s) {
    if (np == 0) return;
    k_soa_to_pairs<<<blocks(np, kThreads), kThreads, 0, s>>>(soa, np, dst);
}

void launch_pairs_to_soa(PState src, int64_t np, double* soa, cudaStream_t s) {
    if (np == 0) return;
    k_pairs_to_soa<<<blocks(np, kThreads), kThreads, 0, s>>>(src, np, soa);
}

void launch_push_key(const Geom& g, PState cur, int64_t np, const uint32_t* offs, const double* E4,
                     int push, uint32_t* key, uint16_t* rank, uint32_t* count, int* err_flag,
                     cudaStream_t s) {
    if (np == 0) return;
    if (push) {
        const unsigned nbrick = (unsigned)(((int64_t)g.n * g.n * g.n) / kBrick);
        k_push_key_brick<<<nbrick, kThreads, 0, s>>>(g, cur, offs, E4, key, rank, count, err_flag);
    } else {
        const unsigned nb = std::min<unsigned>(blocks(np, kThreads), 148u * 32u);
        k_push_key<false><<<nb, kThreads, 0, s>>>(g, cur, np, E4, key, rank, count, err_flag);
    }
}

void launch_keys_only(const Geom& g, PState cur, int64_t np, uint32_t* key, cudaStream_t s) {
    if (np == 0) return;
    k_keys_only<<<blocks(np, kThreads), kThreads, 0, s>>>(g, cur, np, key);
}

size_t scan_scratch_bytes(int64_t ncell) {
    return sizeof(uint32_t) * (size_t)(blocks(ncell, kScanTile) + 1);
}

void launch_scan(const uint32_t* count, uint32_t* offs, int64_t ncell, uint32_t* scratch, cudaStream_t s) {
    const unsigned nb = blocks(ncell, kScanTile);
    k_scan_reduce<<<nb, kThreads, 0, s>>>(count, ncell, scratch);
    k_scan_bsum<<<1, 1024, 0, s>>>(scratch, (int)nb);
    k_scan_apply<<<nb, kThreads, 0, s>>>(count, offs, ncell, scratch);
}

void launch_place(const uint32_t* key, const uint16_t* rank, int64_t np, const uint32_t* offs,
                  uint32_t* perm, cudaStream_t s) {
    if (np == 0) return;
    k_place<<<blocks((np + 3) / 4, kThreads), kThreads, 0, s>>>(key, rank, np, offs, perm);
}

void launch_reorder_deposit(const Geom& g, const uint32_t* offs, const uint32_t* perm, PState cur,
                            PState nxt, int push, double* rho_buf, int* err_flag, cudaStream_t s) {
    const unsigned nbrick = (unsigned)(((int64_t)g.n * g.n * g.n) / kBrick);
    static const int variant = getenv("PIC_REORDER_VARIANT") ? atoi(getenv("PIC_REORDER_VARIANT")) : 3;
    if (variant == 3) {
        if (push)
            k_reorder_deposit_async<true><<<nbrick, kThreads, kReorderAsyncSmem, s>>>(g, offs, perm, cur, nxt, rho_buf, err_flag);
        else
            k_reorder_deposit_async<false><<<nbrick, kThreads, kReorderAsyncSmem, s>>>(g, offs, perm, cur, nxt, rho_buf, err_flag);
        return;
    }
    const bool fs = reorder_frac_smem();
    const size_t sm = reorder_smem(fs);
    static const int kb = getenv("PIC_REORDER_KB") ? atoi(getenv("PIC_REORDER_KB")) : 4;
    if (push && fs && kb == 4)
        k_reorder_deposit<true, true, 4><<<nbrick, kThreads, sm, s>>>(g, offs, perm, cur, nxt, rho_buf, err_flag);
    else if (push && fs && kb == 8)
        k_reorder_deposit<true, true, 8><<<nbrick, kThreads, sm, s>>>(g, offs, perm, cur, nxt, rho_buf, err_flag);
    else if (push && fs)
        k_reorder_deposit<true, true><<<nbrick, kThreads, sm, s>>>(g, offs, perm, cur, nxt, rho_buf, err_flag);
    else if (push)
        k_reorder_deposit<true, false><<<nbrick, kThreads, sm, s>>>(g, offs, perm, cur, nxt, rho_buf, err_flag);
    else if (fs)
        k_reorder_deposit<false, true><<<nbrick, kThreads, sm, s>>>(g, offs, perm, cur, nxt, rho_buf, err_flag);
    else
        k_reorder_deposit<false, false><<<nbrick, kThreads, sm, s>>>(g, offs, perm, cur, nxt, rho_buf, err_flag);
}

void particles_set_smem_limits() {
    cudaFuncSetAttribute(k_reorder_deposit_async<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kReorderAsyncSmem);
    cudaFuncSetAttribute(k_reorder_deposit_async<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kReorderAsyncSmem);
    cudaFuncSetAttribute(k_reorder_deposit<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)reorder_smem(true));
    cudaFuncSetAttribute(k_reorder_deposit<true, true, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)reorder_smem(true));
    cudaFuncSetAttribute(k_reorder_deposit<true, true, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)reorder_smem(true));
    cudaFuncSetAttribute(k_reorder_deposit<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)reorder_smem(true));
    cudaFuncSetAttribute(k_reorder_deposit<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)reorder_smem(false));
    cudaFuncSetAttribute(k_reorder_deposit<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)reorder_smem(false));
}

void launch_sort_segments(const uint32_t* offs, int64_t ncell, uint32_t* perm, cudaStream_t s) {
    k_sort_segments<<<blocks(ncell, kThreads), kThreads, 0, s>>>(offs, ncell, perm);
}

void launch_half_kick(const Geom& g, PState cur, int64_t np, const double* E4, cudaStream_t s) {
    if (np == 0) return;
    k_half_kick<<<blocks(np, kThreads), kThreads, 0, s>>>(g, cur, np, E4);
}

}  // namespace pic
