// particle_kernels.cu -- particle side of the PIC step on sm_100a.
//
// Particle state lives in HBM as three streams of 128-bit pairs (pic_device.cuh):
// (x, y), (z, v_z), (v_x, v_y), sorted by the rank-local Morton cell key (D#14).
// One step (after the solve) is:
//   push_key : one CTA per brick of 256 cells: stage the brick's E node tile in
//              shared memory, stream the brick's particles, gather E (CIC), kick v
//              in place, drift to x' (not stored), key of the new cell and its
//              arrival rank (count atomic).  P > 1: particles whose new cell lies in
//              another slab go to that rank's send buffer (x', v', old global key,
//              old index) instead.
//   [P > 1: counts all-to-all, payload send/recv, arrivals keyed and counted]
//   scan     : offs = exclusive scan of the cell counts.
//   place    : perm[offs[key] + rank] = i (no atomics).
//   reorder_deposit : one CTA per brick: the stable order inside each cell (D#14),
//              the particles gathered through perm with cp.async straight into
//              their sorted slots in shared memory, the drift recomputed
//              bit-identically from the stored v', x' v' streamed out coalesced,
//              and the CIC charge summed per cell in stable order, folded into a
//              node tile in shared memory and flushed with one fp64 RED.ADD per node.
#include <algorithm>
#include <cstdlib>

#include "kernels.h"

// PIC_PLACE_ATOMIC: 1 = the cell count of the push is a fire-and-forget reduction (RED: no
// returned rank to wait for) and place takes each particle's position from a cursor per
// cell (the scan leaves offs in `count`, place does atomicAdd on it); 0 (default) = the
// push's count atomics return the arrival ranks (stored, 2 B per particle; issued in
// batches so their round trips overlap) and place reads offs[key] + rank.  Both give the
// same per-cell multiset of positions; the stable order inside a cell is restored by
// reorder_deposit either way.  r02 at 512^3: 1 moved the atomic latency from push_key
// (19.9 -> 16.3 ms) into place (7.1 -> 10.3 ms), a net loss.
#ifndef PIC_PLACE_ATOMIC
#define PIC_PLACE_ATOMIC 0
#endif
// PIC_PLACE_AGG (with PIC_PLACE_ATOMIC=1, P = 1): place takes its cursor positions per source
// brick -- a shared-memory histogram of the brick's particles over the window around it
// (AggWin) and one returned cursor atomic per non-empty window cell -- instead of one
// returned atomic per particle.
#ifndef PIC_PLACE_AGG
#define PIC_PLACE_AGG 0
#endif
#ifndef PIC_ATOM_BATCH      // particles per batch of returned count atomics in push_key
#define PIC_ATOM_BATCH 1        // r02 A/B at 512^3: 1, 2, 4, 8 -> 19.97, 20.21, 20.19, 19.94 ms
#endif
// PIC_PK_AGG: 1 = push_key (P = 1) counts arrivals per brick first: a shared-memory histogram
// over a window around the brick (AggWin) gives each particle its rank among the brick's
// arrivals in that cell, then one returned global atomic per non-empty window cell
// reserves the brick's block of arrival ranks (about half as many global atomics as
// particles); particles landing outside the window take one global atomic each as before.
// Measured (r02, 512^3): push_key 20.7 vs 20.0 ms -- the shared histogram, the second
// pass and the extra barriers cost more than the halved returned atomics save.  Off.
#ifndef PIC_PK_AGG
#define PIC_PK_AGG 0
#endif

namespace pic {

namespace {

constexpr int kThreads = 256;
constexpr int kBrick = 256;     // cells per brick (Morton 8 bits: 8 x 8 x 4)
constexpr uint32_t kNoKey = 0xffffffffu;

// ---------------------------------------------------------------- init -----
// Landau initial condition: x_d by Newton on the inverse CDF of
// (1 + alpha cos(k x))/L from x = u_d L (|dx| < 1e-12 or 32 iterations),
// velocities by Box-Muller from u_3..u_6, Philox counter = global particle index
// (D#10).
__device__ __forceinline__ void uniforms(uint64_t j, uint32_t s0, uint32_t s1, double u[8]) {
#pragma unroll
    for (int b = 0; b < 4; ++b) {
        uint32_t c[4] = {(uint32_t)j, (uint32_t)(j >> 32), (uint32_t)b, 0u};
        philox4x32_10(c, s0, s1);
        const uint64_t w0 = (uint64_t)c[0] | ((uint64_t)c[1] << 32);
        const uint64_t w1 = (uint64_t)c[2] | ((uint64_t)c[3] << 32);
        u[2 * b] = (double)(w0 >> 11) * 0x1p-53;
        u[2 * b + 1] = (double)(w1 >> 11) * 0x1p-53;
    }
}

__device__ __forceinline__ double landau_x(const Geom& g, double u, double k, double alpha) {
    const double ak = alpha / k;
    const double target = u * g.L;
    double xx = target;
    for (int it = 0; it < 32; ++it) {
        const double F = __dsub_rn(__dadd_rn(xx, __dmul_rn(ak, sin(k * xx))), target);
        const double dF = __dadd_rn(1.0, __dmul_rn(alpha, cos(k * xx)));
        const double dx = __ddiv_rn(F, dF);
        xx = __dsub_rn(xx, dx);
        if (fabs(dx) < 1e-12) break;
    }
    return wrap(xx, g.L);
}

__device__ __forceinline__ void landau_particle(const Geom& g, const double u[8], double k,
                                                double alpha, double x[3], double v[3]) {
    for (int d = 0; d < 3; ++d) x[d] = landau_x(g, u[d], k, alpha);
    const double two_pi = 6.283185307179586476925286766559;
    const double r1 = sqrt(-2.0 * log(1.0 - u[3]));
    const double r2 = sqrt(-2.0 * log(1.0 - u[5]));
    v[0] = r1 * cos(two_pi * u[4]);
    v[1] = r1 * sin(two_pi * u[4]);
    v[2] = r2 * cos(two_pi * u[6]);
}

// Ownership of particle j at P > 1 from its y and z only (u_1, u_2): slabs need z alone.
__device__ __forceinline__ bool owns_yz(const Geom& g, const double u[8], double k, double alpha) {
    const int iz = cell_of(__dmul_rn(landau_x(g, u[2], k, alpha), g.inv_h), g.n);
    if (iz < g.z0 || iz >= g.z0 + g.nzl) return false;
    if (g.Py == 1) return true;
    const int iy = cell_of(__dmul_rn(landau_x(g, u[1], k, alpha), g.inv_h), g.n);
    return iy >= g.y0 && iy < g.y0 + g.nyl;
}

// P = 1: particle j at index j.
__global__ void __launch_bounds__(kThreads) k_sample(Geom g, PState st, int64_t np, double k,
                                                     double alpha, uint32_t s0, uint32_t s1) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= np) return;
    double u[8], x[3], v[3];
    uniforms((uint64_t)j, s0, s1, u);
    landau_particle(g, u, k, alpha, x, v);
    store_particle(st, j, x, v);
}

// P > 1, pass 1: owned particles of each block of 256 global indices (only z is
// needed to decide ownership).
__global__ void __launch_bounds__(kThreads) k_sample_count(Geom g, int64_t npg, double k, double alpha,
                                                           uint32_t s0, uint32_t s1,
                                                           uint32_t* __restrict__ bcount) {
    __shared__ uint32_t red[kThreads / 32];
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    bool own = false;
    if (j < npg) {
        double u[8];
        uniforms((uint64_t)j, s0, s1, u);
        own = owns_yz(g, u, k, alpha);
    }
    const uint32_t b = __popc(__ballot_sync(0xffffffffu, own));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = b;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t t = 0;
        for (int w = 0; w < kThreads / 32; ++w) t += red[w];
        bcount[blockIdx.x] = t;
    }
}

// P > 1, pass 2: the owned particles written in ascending global index (the
// oracle's initial order restricted to the slab, SURVEY c.1 Init 4).
__global__ void __launch_bounds__(kThreads) k_sample_write(Geom g, PState st, int64_t npg, double k,
                                                           double alpha, uint32_t s0, uint32_t s1,
                                                           const uint32_t* __restrict__ boffs) {
    __shared__ uint32_t wpre[kThreads / 32];
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    double u[8];
    bool own = false;
    if (j < npg) {
        uniforms((uint64_t)j, s0, s1, u);
        own = owns_yz(g, u, k, alpha);
    }
    const unsigned bal = __ballot_sync(0xffffffffu, own);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) wpre[wid] = __popc(bal);
    __syncthreads();
    uint32_t pre = 0;
    for (int w = 0; w < wid; ++w) pre += wpre[w];
    if (own) {
        const int64_t o = (int64_t)boffs[blockIdx.x] + pre + __popc(bal & ((1u << lane) - 1u));
        double x[3], v[3];
        landau_particle(g, u, k, alpha, x, v);
        store_particle(st, o, x, v);
    }
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

// ----------------------------------------------------------- key (import) ---
// Particles in any order (init, pic_set_particles, re-deposit): key of the current
// position, rank = count[key]++.  A position outside [0, L) or outside the slab
// sets err[1].
__global__ void __launch_bounds__(kThreads) k_key_import(Geom g, PState cur, int64_t np,
                                                         uint32_t* __restrict__ key,
                                                         uint16_t* __restrict__ rank,
                                                         uint32_t* __restrict__ count,
                                                         int* __restrict__ err) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < np; i += stride) {
        double x[3], v[3];
        load_particle(cur, i, x, v);
        // an invalid position is reported (err[1]) and replaced by a valid one inside
        // the slab, so the state stays consistent for every later kernel
        bool bad = false;
#pragma unroll
        for (int d = 0; d < 3; ++d)
            if (!(x[d] >= 0.0 && x[d] < g.L)) { x[d] = 0.0; bad = true; }
        int iz = 0, iy = 0;
        uint32_t k = key_of(g, x, &iz, &iy);
        if (!in_domain(g, iy, iz)) {
            x[1] = ((double)g.y0 + 0.5) / g.inv_h;
            x[2] = ((double)g.z0 + 0.5) / g.inv_h;
            k = key_of(g, x, &iz, &iy);
            bad = true;
        }
        if (bad) {
            atomicExch(err + 1, 1);
            store_particle(cur, i, x, v);
        }
        key[i] = k;
        if (PIC_PLACE_ATOMIC) {
            atomicAdd(count + k, 1u);
        } else {
            const uint32_t r = atomicAdd(count + k, 1u);
            if (r > 0xffffu) atomicExch(err, 1);
            rank[i] = (uint16_t)r;
        }
    }
}

// ----------------------------------------------------------- push + key ----
// The step's push: one CTA per brick.  The brick's particles
// are the contiguous sorted range [offs[c0], offs[c0 + 256)) and all their CIC
// corners lie in the brick's 9 x 9 x 5 node tile (slab planes bz .. bz + 4, the
// last possibly the halo), staged in shared memory; the gather reads it with the
// same weights, corner order and fma chain as the oracle (D#17).  Kick v in place,
// drift to x' (not stored), key, rank.  Leavers (P > 1) are 64-B records (x', y'),
// (z', vz'), (vx', vy'), (old global key | old index << 32), staged per brick in
// shared memory, then written either into this rank's send segment of their
// destination (NCCL transport) or, with peer memory, straight into the
// destination's receive buffer at slots from its arrival counter (one system-scope
// atomic per brick and destination over NVLink).
struct SendBuf {
    double2* data;        // segment r at data + 4 * segs.off[r]
    uint32_t* count;      // [P] leavers per destination (both transports)
    SendSegs segs;
    PeerRecv peers;
    int remote;           // 1: peer-memory transport
};

// Slot base for n leavers to destination dr; their records go to dst_rec(dr, slot).
__device__ __forceinline__ uint32_t leave_reserve(const SendBuf& sb, int dr, uint32_t n) {
    if (!sb.remote) return atomicAdd(sb.count + dr, n);
    atomicAdd(sb.count + dr, n);
    return (uint32_t)atomicAdd_system(sb.peers.peer_arr[dr], (unsigned long long)n);
}
__device__ __forceinline__ double2* leave_rec(const SendBuf& sb, int dr, uint32_t slot) {
    if (!sb.remote) return slot < (uint32_t)sb.segs.cap[dr] ? sb.data + (sb.segs.off[dr] + slot) * 4 : nullptr;
    return slot < (uint64_t)sb.peers.recv_cap ? sb.peers.peer_recv[dr] + (int64_t)slot * 4 : nullptr;
}

// Leavers staged per brick before one atomic per destination.  A brick on a slab face
// loses ~20% of its ~2048 particles per step (the thermal displacement is ~2 cells against
// a 4-cell brick), so 128 slots overflowed on every face brick and the overflow took one
// global atomic per particle on a single counter per destination (r02: the P > 1 push_key
// cost +55% per particle at P = 4).  320 slots plus a warp-aggregated overflow.
constexpr int kLeaveCap = 320;

// Arrival window of a brick (PIC_PK_AGG): its 8 x 8 x 4 cells +- 4 in x and y and +- 3 in z
// (2560 cells).  With the thermal displacement of ~2 cells per step about 7% of the particles
// land outside.  Shared memory per CTA: the count and the key of each window cell (20 KB)
// and the (bin, rank in bin) of the brick's first kInfoCap particles (9 KB), beside the
// 17 KB E tile: 4 CTAs per SM.  P > 1 keeps the direct count atomics (the leaver staging
// uses that shared memory).
struct AggWin {
    static constexpr int H = 4, HZ = 3, WX = 8 + 2 * H, WY = 8 + 2 * H, WZ = 4 + 2 * HZ, NB = WX * WY * WZ;
    // bin of local cell (ix, iyl, izl) for the brick at (bx, by, bz), -1 outside the window;
    // coordinates wrap where the rank's domain spans the whole periodic dimension
    static __device__ __forceinline__ int bin(const Geom& g, int ix, int iyl, int izl, int bx, int by, int bz) {
        const int dx = (ix - bx + H) & g.nmask;
        int dy = iyl - by + H, dz = izl - bz + HZ;
        if (g.nyl == g.n) dy &= g.nmask;
        if (g.nzl == g.n) dz &= g.nmask;
        if ((unsigned)dx >= (unsigned)WX || (unsigned)dy >= (unsigned)WY || (unsigned)dz >= (unsigned)WZ) return -1;
        return (dz * WY + dy) * WX + dx;
    }
};
constexpr int kInfoCap = 2304;      // particles per brick with a shared (bin, rank) record

template <bool MR>
__global__ void __launch_bounds__(kThreads, MR ? 3 : 4) k_push_key_brick(Geom g, PState cur,
                                                             const uint32_t* __restrict__ offs,
                                                             const double* __restrict__ E4,
                                                             uint32_t* __restrict__ key,
                                                             uint16_t* __restrict__ rank,
                                                             uint32_t* __restrict__ count,
                                                             SendBuf sb, uint32_t* __restrict__ bprev,
                                                             int* __restrict__ err) {
    // E tile in x-pairs: entry (z, y, x) = (E_d(x), E_d(x + 1)) for d = x, y, z, so the two
    // x corners of one (y, z) corner pair are three 16-B shared loads (48 B) instead of two
    // 32-B node records (64 B): a quarter less shared-memory traffic per particle
    // (ncu r01: the kernel ran at 79% of the L1/shared throughput)
    __shared__ double2 ptile[5 * 9 * 8][3];
    __shared__ double2 lbuf[MR ? kLeaveCap : 1][4];      // leavers of this brick (P > 1)
    __shared__ uint8_t ldst[MR ? kLeaveCap : 1];
    __shared__ uint32_t lcount[8], lbase[8], nleave;
    constexpr bool kAgg = PIC_PK_AGG && !PIC_PLACE_ATOMIC && PIC_ATOM_BATCH == 1 && !MR;
    using Win = AggWin;
    __shared__ uint32_t hist[kAgg ? Win::NB : 1], binkey[kAgg ? Win::NB : 1];
    __shared__ uint32_t info[kAgg ? kInfoCap : 1];      // bin | rank in bin << 12, ~0: no record
    const int t = threadIdx.x;
    const uint32_t c0 = blockIdx.x * kBrick;
    int bx, by, bz;
    unlkey(g, c0, bx, by, bz);    // bz: slab plane
    for (int q = t; q < 9 * 9 * 5; q += kThreads) {
        const int nx = q % 9, ny = (q / 9) % 9, nz = q / 81;
        const int64_t m = ((int64_t)(bz + nz) * g.nyr + yrow(g, by + ny)) * g.n + ((bx + nx) & g.nmask);
        double ex, ey, ez;
        ldg_node(E4 + 4 * m, ex, ey, ez);
        const int row = (nz * 9 + ny) * 8;
        if (nx < 8) {
            ptile[row + nx][0].x = ex;
            ptile[row + nx][1].x = ey;
            ptile[row + nx][2].x = ez;
        }
        if (nx > 0) {
            ptile[row + nx - 1][0].y = ex;
            ptile[row + nx - 1][1].y = ey;
            ptile[row + nx - 1][2].y = ez;
        }
    }
    if (t < 8) lcount[t] = 0;
    if (t == 0) nleave = 0;
    if (kAgg)
        for (int b = t; b < Win::NB; b += kThreads) hist[b] = 0;
    const uint32_t P0 = __ldg(offs + c0), P1 = __ldg(offs + c0 + kBrick);
    if (bprev && t == 0) {        // this order's brick ranges, for the reorder's L2 prefetch
        bprev[blockIdx.x] = P0;
        if (blockIdx.x == gridDim.x - 1) bprev[gridDim.x] = P1;
    }
    __syncthreads();
    double xn[3], vn[3];
    if (P0 + t < P1) load_particle(cur, P0 + t, xn, vn);
    // The count atomics return each particle's arrival rank; with PIC_ATOM_BATCH > 1 they are
    // issued in batches after the batch's pushes so their round trips overlap.  Measured
    // without gain: the cost of the returned rank is the L2 atomic itself (a fire-and-forget
    // RED count made push_key 3.6 ms faster, see PIC_PLACE_ATOMIC), not its exposed latency.
    constexpr int kAtomBatch = PIC_PLACE_ATOMIC ? 1 : PIC_ATOM_BATCH;
    for (uint32_t i0 = P0 + t; i0 < P1; i0 += kAtomBatch * kThreads) {
        uint32_t kq[kAtomBatch];
#pragma unroll
        for (int u = 0; u < kAtomBatch; ++u) {
            const uint32_t i = i0 + u * kThreads;
            kq[u] = kNoKey;
            if (i >= P1) continue;
            double x[3] = {xn[0], xn[1], xn[2]}, v[3] = {vn[0], vn[1], vn[2]};
            // next particle's loads in flight while this one is pushed
            if (i + kThreads < P1) load_particle(cur, i + kThreads, xn, vn);
            const double x0 = x[0], y0 = x[1], z0 = x[2];
            int ii[3];
            double w[3][2];
            cic_weights(g, x, ii, w);
            const int lx = ii[0] - bx, ly = ii[1] - g.y0 - by, lz = ii[2] - g.z0 - bz;
            double e0 = 0.0, e1 = 0.0, e2 = 0.0;
#pragma unroll
            for (int c = 0; c < 2; ++c)
#pragma unroll
                for (int b = 0; b < 2; ++b) {
                    const double2* pe = ptile[((lz + c) * 9 + (ly + b)) * 8 + lx];
                    const double2 px = pe[0], py = pe[1], pz = pe[2];
                    const double wt0 = __dmul_rn(__dmul_rn(w[0][0], w[1][b]), w[2][c]);
                    const double wt1 = __dmul_rn(__dmul_rn(w[0][1], w[1][b]), w[2][c]);
                    e0 = __fma_rn(wt0, px.x, e0);          // corner order z, y, x (x inner): a = 0 ...
                    e1 = __fma_rn(wt0, py.x, e1);
                    e2 = __fma_rn(wt0, pz.x, e2);
                    e0 = __fma_rn(wt1, px.y, e0);          // ... then a = 1, as the oracle (D#17)
                    e1 = __fma_rn(wt1, py.y, e1);
                    e2 = __fma_rn(wt1, pz.y, e2);
                }
            double ep[3] = {e0, e1, e2};
            kick(g, ep, v);
            drift(g, x, v);
            st_zv(cur.zv + 2 * i, make_double2(z0, v[2]), make_double2(v[0], v[1]));   // kicked v in place
            int iz, iy, ix;
            const uint32_t k = key_of(g, x, &iz, &iy, &ix);
            if (MR && !in_domain(g, iy, iz)) {   // leaver: staged, sent below
                const int dr = owner_of(g, iy, iz);
                const double xo[3] = {x0, y0, z0};
                const uint32_t oldg = gkey_of(g, xo);           // its tie key (D#15)
                const double2 p0 = make_double2(x[0], x[1]), p1 = make_double2(x[2], v[2]),
                              p2 = make_double2(v[0], v[1]),
                              p3 = make_double2(__longlong_as_double((long long)((uint64_t)oldg | ((uint64_t)i << 32))), 0.0);
                const uint32_t s = atomicAdd(&nleave, 1u);
                if (s < (uint32_t)kLeaveCap) {
                    lbuf[s][0] = p0; lbuf[s][1] = p1; lbuf[s][2] = p2; lbuf[s][3] = p3;
                    ldst[s] = (uint8_t)dr;
                    atomicAdd(&lcount[dr], 1u);
                } else {      // staging full: straight to the global buffer, one reserve per warp and destination
                    const unsigned grp = __match_any_sync(__activemask(), dr);
                    const int lead = __ffs(grp) - 1, lane = threadIdx.x & 31;
                    uint32_t base = 0;
                    if (lane == lead) base = leave_reserve(sb, dr, (uint32_t)__popc(grp));
                    base = __shfl_sync(grp, base, lead) + (uint32_t)__popc(grp & ((1u << lane) - 1u));
                    double2* d = leave_rec(sb, dr, base);
                    if (d) {
                        d[0] = p0; d[1] = p1; d[2] = p2; d[3] = p3;
                    } else {
                        atomicExch(err + 2, 1);
                    }
                }
                key[i] = kNoKey;
                continue;
            }
            key[i] = k;
            if (kAgg) {       // rank among the brick's arrivals in the cell, offset below
                const uint32_t li = i - P0;
                const int b = li < (uint32_t)kInfoCap ? Win::bin(g, ix, iy - g.y0, iz - g.z0, bx, by, bz) : -1;
                if (b >= 0) {
                    const uint32_t lr = atomicAdd(&hist[b], 1u);
                    if (lr == 0) binkey[b] = k;
                    info[li] = (uint32_t)b | (lr << 12);
                } else {
                    const uint32_t r = atomicAdd(count + k, 1u);
                    if (r > 0xffffu) atomicExch(err, 1);
                    rank[i] = (uint16_t)r;
                    if (li < (uint32_t)kInfoCap) info[li] = ~0u;
                }
            } else if (PIC_PLACE_ATOMIC) {
                atomicAdd(count + k, 1u);          // RED: nothing to wait for
            } else {
                kq[u] = k;
            }
        }
        if (!PIC_PLACE_ATOMIC && !kAgg) {
            uint32_t rq[kAtomBatch];
#pragma unroll
            for (int u = 0; u < kAtomBatch; ++u) rq[u] = kq[u] != kNoKey ? atomicAdd(count + kq[u], 1u) : 0u;
#pragma unroll
            for (int u = 0; u < kAtomBatch; ++u)
                if (kq[u] != kNoKey) {
                    if (rq[u] > 0xffffu) atomicExch(err, 1);
                    rank[i0 + u * kThreads] = (uint16_t)rq[u];
                }
        }
    }
    if (kAgg) {    // one returned global atomic per non-empty window cell: the brick's base rank
        __syncthreads();
        constexpr int kPer = (Win::NB + kThreads - 1) / kThreads;
        uint32_t cb[kPer], rb[kPer];      // all of this thread's bins' atomics in flight at once
#pragma unroll
        for (int u = 0; u < kPer; ++u) {
            const int b = t + u * kThreads;
            cb[u] = b < Win::NB ? hist[b] : 0u;
        }
#pragma unroll
        for (int u = 0; u < kPer; ++u)
            if (cb[u]) rb[u] = atomicAdd(count + binkey[t + u * kThreads], cb[u]);
#pragma unroll
        for (int u = 0; u < kPer; ++u)
            if (cb[u]) hist[t + u * kThreads] = rb[u];
        __syncthreads();
        const uint32_t Pe = min(P1, P0 + (uint32_t)kInfoCap);
        for (uint32_t i = P0 + t; i < Pe; i += kThreads) {
            const uint32_t v = info[i - P0];
            if (v == ~0u) continue;
            const uint32_t r = hist[v & 0xfffu] + (v >> 12);
            if (r > 0xffffu) atomicExch(err, 1);
            rank[i] = (uint16_t)r;
        }
    }
    if (MR) {      // one global atomic per destination, then the staged payloads
        __syncthreads();
        if (t < g.P) {
            lbase[t] = lcount[t] ? leave_reserve(sb, t, lcount[t]) : 0u;
            lcount[t] = 0;
        }
        __syncthreads();
        const int nl = min((int)nleave, kLeaveCap);
        for (int s = t; s < nl; s += kThreads) {
            const int dr = ldst[s];
            double2* d = leave_rec(sb, dr, lbase[dr] + atomicAdd(&lcount[dr], 1u));
            if (d) {
                d[0] = lbuf[s][0]; d[1] = lbuf[s][1]; d[2] = lbuf[s][2]; d[3] = lbuf[s][3];
            } else {
                atomicExch(err + 2, 1);
            }
        }
        if (sb.remote && nleave) __threadfence_system();   // peer stores done before the barrier
    }
}

// Arrivals (P > 1): key and rank of each received particle, at extended index
// n_old + a (the permutation addresses cur below n_old and the receive buffer above).
__global__ void __launch_bounds__(kThreads) k_key_arrivals(Geom g, const double2* __restrict__ recv,
                                                           int64_t narr, int64_t n_old,
                                                           uint32_t* __restrict__ key,
                                                           uint16_t* __restrict__ rank,
                                                           uint32_t* __restrict__ count,
                                                           int* __restrict__ err,
                                                           const unsigned long long* __restrict__ dcnt) {
    if (dcnt) {          // peer-memory transport: counts on the device (narr = capacity)
        narr = min((int64_t)dcnt[DC_ARR], narr);
        n_old = (int64_t)dcnt[DC_N];
    }
    for (int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; a < narr;
         a += (int64_t)gridDim.x * blockDim.x) {
        const double2 p0 = recv[4 * a], p1 = recv[4 * a + 1];
        const double x[3] = {p0.x, p0.y, p1.x};
        int iz, iy;
        uint32_t k = key_of(g, x, &iz, &iy);
        if (!in_domain(g, iy, iz)) { atomicExch(err + 1, 1); k = 0; }
        key[n_old + a] = k;
        if (PIC_PLACE_ATOMIC) {
            atomicAdd(count + k, 1u);
        } else {
            const uint32_t r = atomicAdd(count + k, 1u);
            if (r > 0xffffu) atomicExch(err, 1);
            rank[n_old + a] = (uint16_t)r;
        }
    }
}

// Peer-memory transport: n <- n - leavers + arrivals after the step's sort.
__global__ void k_counts_update(int P, unsigned long long* dcnt, const uint32_t* __restrict__ send_count,
                                int64_t np_cap, int* err) {
    unsigned long long leave = 0;
    for (int r = 0; r < P; ++r) leave += send_count[r];
    const unsigned long long n = dcnt[DC_N] - leave + dcnt[DC_ARR];
    if ((int64_t)n > np_cap) atomicExch(err + 2, 1);
    dcnt[DC_N] = n;
    dcnt[DC_LEAVE] = leave;
    dcnt[DC_MIGRATED] += leave;
    dcnt[DC_ARR] = 0;
}

__global__ void k_set_u64(unsigned long long* p, unsigned long long v) { *p = v; }

// Peer-memory migration, batched (default): push_key staged the leavers in this rank's
// local send segments; one thread per destination reserves a contiguous range of the
// destination's receive buffer (one system-scope atomic per rank pair) ...
__global__ void k_leaver_reserve(int P, int rank, const uint32_t* __restrict__ send_count, PeerRecv peers,
                                 const SendSegs segs, uint32_t* __restrict__ base, int* err) {
    const int r = threadIdx.x;
    if (r >= P || r == rank) return;
    const uint32_t n = min(send_count[r], (uint32_t)segs.cap[r]);
    base[r] = 0;
    if (n == 0) return;
    const unsigned long long b = atomicAdd_system(peers.peer_arr[r], (unsigned long long)n);
    if (b + n > (unsigned long long)peers.recv_cap) atomicExch(err + 2, 1);
    base[r] = (uint32_t)b;
}
// ... and every CTA streams its share of the records over NVLink with coalesced 16-B
// stores (the per-brick remote atomics and 64-B stores of the unbatched path ran at
// ~0.1 TB/s and cost 2-3 ms per step at 512^3 on 2-4 GPUs).
__global__ void __launch_bounds__(256) k_leaver_copy(int P, int rank, const double2* __restrict__ send,
                                                     const SendSegs segs, const uint32_t* __restrict__ send_count,
                                                     const uint32_t* __restrict__ base, PeerRecv peers) {
    for (int r = 0; r < P; ++r) {
        if (r == rank) continue;
        const int64_t n = min(send_count[r], (uint32_t)segs.cap[r]);
        const int64_t b = base[r];
        const int64_t m = n < peers.recv_cap - b ? n : peers.recv_cap - b;
        const double2* src = send + 4 * segs.off[r];
        double2* dst = peers.peer_recv[r] + 4 * b;
        for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < 4 * m;
             i += (int64_t)gridDim.x * blockDim.x)
            dst[i] = __ldcs(src + i);
    }
    __threadfence_system();
}

__global__ void __launch_bounds__(kThreads) k_gkeys(Geom g, PState cur, int64_t np,
                                                    uint32_t* __restrict__ key) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= np) return;
    double x[3], v[3];
    load_particle(cur, i, x, v);
    key[i] = gkey_of(g, x);
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

__global__ void __launch_bounds__(kThreads) k_scan_apply(uint32_t* __restrict__ count,
                                                         uint32_t* __restrict__ offs, int64_t ncell,
                                                         const uint32_t* __restrict__ bsum, int cursor) {
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
        uint4* pc = reinterpret_cast<uint4*>(count + base);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const uint4 o = make_uint4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
            po[q] = o;
            if (cursor) pc[q] = o;          // the counts become the place cursors (offs)
        }
    } else {
        for (int q = 0; q < 16; ++q)
            if (base + q < ncell) {
                offs[base + q] = v[q];
                if (cursor) count[base + q] = v[q];
            }
    }
    if (ncell > base && ncell <= base + 16) offs[ncell] = run;   // owner of the last cell: total
}

// ----------------------------------------------------------------- place ---
// perm[offs[key[i]] + rank[i]] = i  (no atomics: ranks came from the count atomic);
// leavers (key = kNoKey) are skipped.
__global__ void __launch_bounds__(kThreads) k_place(const uint32_t* __restrict__ key,
                                                    const uint16_t* __restrict__ rank, int64_t np,
                                                    uint32_t* __restrict__ offs,
                                                    uint32_t* __restrict__ perm,
                                                    const unsigned long long* __restrict__ dcnt,
                                                    int64_t cap, int* __restrict__ err) {
    // peer-memory transport: the entry count is on the device, and a sorted position
    // beyond the arrays (a slab over capacity) is dropped and flagged
    if (dcnt) np = min(np, (int64_t)(dcnt[DC_N] + dcnt[DC_ARR]));
    // Consecutive lanes take consecutive particles (four strided passes per CTA), so a
    // warp's 32 perm stores land in the ~4 cells those particles arrive in: a handful of
    // 32-B sectors per store instruction instead of ~16 with four particles per thread
    // (ncu: the old mapping was L2-request bound at 74% L2 throughput, 1.6 TB/s DRAM).
    const int64_t base = (int64_t)blockIdx.x * (4 * kThreads) + threadIdx.x;
    uint32_t k[4], r[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int64_t i = base + q * kThreads;
        k[q] = i < np ? __ldg(key + i) : kNoKey;
        r[q] = (i < np && !PIC_PLACE_ATOMIC) ? __ldg(rank + i) : 0u;
    }
    uint32_t pos[4];
#pragma unroll
    for (int q = 0; q < 4; ++q)
        pos[q] = k[q] == kNoKey ? 0u : (PIC_PLACE_ATOMIC ? atomicAdd(offs + k[q], 1u) : __ldg(offs + k[q]) + r[q]);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        if (k[q] == kNoKey) continue;
        if (pos[q] < (uint64_t)cap) perm[pos[q]] = (uint32_t)(base + q * kThreads);
        else atomicExch(err + 2, 1);
    }
}

// Node tile of a brick: 9 x 9 x 5 nodes, slab planes bz .. bz + 4 (the last one
// possibly the ghost plane nzl); x and y wrap periodically (pencils: local rows, the last
// one the ghost row).  Rows are kTileRow = 10 doubles apart so each starts 16-B aligned.
constexpr int kTileRow = 10;
constexpr int kTileSize = 5 * 9 * kTileRow;
#ifndef PIC_RD_BULK      // r02 A/B at 512^3: 29.09 ms with the bulk row flush, 28.71 with atomics
#define PIC_RD_BULK 0
#endif

__device__ __forceinline__ void bulk_add_f64(double* gdst, const double* ssrc, unsigned bytes) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(ssrc);
    asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f64 [%0], [%1], %2;"
                 ::"l"(gdst), "r"(s), "r"(bytes) : "memory");
}

__device__ __forceinline__ void fold_flush(const Geom& g, double* tile, const double acc[8], int t,
                                           int bx, int by, int bz, double* __restrict__ rho,
                                           double* ghost) {
    const int lx = (int)compact3((uint32_t)t), ly = (int)compact3((uint32_t)t >> 1),
              lz = (int)compact3((uint32_t)t >> 2);
    // local destinations (one GPU, pencils, or the slabs' own ghost plane): each tile row's
    // first 8 nodes (64 B, 16-B aligned in shared and global memory) go out as one bulk
    // fp64 reduction (UBLKRED: 45 per brick instead of 360 atomics), the 9th as an atomic
    const bool bulk = PIC_RD_BULK && (g.P == 1 || g.Py > 1 || ghost == rho + (int64_t)g.nzl * g.nyr * g.rp);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const int a = q & 1, b = (q >> 1) & 1, c = q >> 2;
        tile[((lz + c) * 9 + (ly + b)) * kTileRow + (lx + a)] += acc[q];
        if (bulk && q == 7) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
    }
    if (bulk) {
        if (t < 45) {
            const int ny = t % 9, nz = t / 9;
            const int iy = yrow(g, by + ny), iz = bz + nz;
            double* row = (g.Py == 1 && iz == g.nzl) ? ghost + gidx(g, 0, iy, 0) : rho + gidx(g, 0, iy, iz);
            const double* trow = tile + t * kTileRow;
            bulk_add_f64(row + bx, trow, 64);
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            const double v8 = trow[8];
            if (v8 != 0.0) atomicAdd(row + ((bx + 8) & g.nmask), v8);
            asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
        }
        return;
    }
    for (int q = t; q < 9 * 9 * 5; q += kThreads) {
        const int nx = q % 9, ny = (q / 9) % 9, nz = q / 81;
        const double val = tile[(nz * 9 + ny) * kTileRow + nx];
#ifdef PIC_RD_SKIP_FLUSH     // diagnostics only (no charge): the cost of the global flush
        if (val != 12345.0) continue;
#endif
        if (val == 0.0) continue;
        const int ix = (bx + nx) & g.nmask, iy = yrow(g, by + ny), iz = bz + nz;
        if (g.Py > 1) {                     // pencils: the local grid holds the ghost row and
            atomicAdd(rho + gidx(g, ix, iy, iz), val);   // plane; folded into the neighbours after
            continue;
        }
        if (iz == g.nzl) {                  // node plane of the next slab (or own plane 0, P = 1)
            if (g.P > 1) atomicAdd_system(ghost + gidx(g, ix, iy, 0), val);
            else atomicAdd(ghost + gidx(g, ix, iy, 0), val);
        } else if (iz == 0 && g.P > 1) {    // shared with the previous slab's ghost adds
            atomicAdd_system(rho + gidx(g, ix, iy, 0), val);
        } else {
            atomicAdd(rho + gidx(g, ix, iy, iz), val);
        }
    }
}

// Corner weight sums of one cell's particles: acc[q] += (w_x w_y) w_z, the last
// product fused into the sum (the charge is compared to a tolerance, D#17 binds
// only the gather and push).
__device__ __forceinline__ void cic_acc(const Geom& g, const double x[3], double acc[8]) {
    int ii[3];
    double w[3][2];
    cic_weights(g, x, ii, w);
    double wxy[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) wxy[q] = __dmul_rn(w[0][q & 1], w[1][q >> 1]);
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[q] = __fma_rn(wxy[q & 3], w[2][q >> 2], acc[q]);
}

// Largest cb with soffs[cb] - soffs[ca] <= cap (uniform across the CTA).
__device__ __forceinline__ int chunk_end(const uint32_t* soffs, int ca, int cap) {
    int lo = ca + 1, hi = kBrick;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (soffs[mid] - soffs[ca] <= (uint32_t)cap) lo = mid; else hi = mid - 1;
    }
    return lo;
}

// ------------------------------------------------------ reorder + deposit --
// Ties inside a cell by pre-sort index (D#14).  The gather is cp.async (LDGSTS,
// 16 B, L2 only) straight into the particle's stable slot of the staged chunk.
// MR (P > 1): entries e >= n_old are arrivals (receive buffer, already drifted by
// their sender); the index rank puts them after the residents of their cell, and
// a fix-up pass re-sorts the (few) cells holding arrivals by (old global key, old
// index) -- the order of the single-domain oracle's global stable sort (D#15).
// Chunk capacity (particles staged per pass; a brick holds ~ppc * 256): 1344 lets
// three CTAs share an SM, which measured faster than two with whole-brick chunks.
#ifndef PIC_RD_CAP
#define PIC_RD_CAP 1344
#endif
#ifndef PIC_RD_MINB
#define PIC_RD_MINB 3
#endif
// PIC_RD_PF: L2 prefetch distance in bricks (0 = off, the default).  The gather's sources are
// the particles of the neighbouring bricks in the previous order (the thermal displacement
// is ~2 cells), ~94% of them within +-1000 bricks in Morton order at 512^3.  Brick b
// prefetches the previous order's particles of brick b + PIC_RD_PF into L2 (two bulk TMA
// prefetches, or per-thread line prefetches with PIC_RD_PF_MODE=1), so that DRAM reads the
// sources as one sequential stream ahead of the gather wavefront.  Measured (r02, ncu at
// 512^3): at 256..2048 bricks ahead the prefetched lines are gone before the gather
// (DRAM reads 73 -> 122..128 GB, +2.8 ms); at 64 ahead they are mostly used (DRAM reads
// 80.7 GB, so ~60% of the gather bytes came from the prefetch) and the kernel is still
// not faster (29.5 vs 28.4 ms): the scattered gather is bound on the L2 side, not by the
// DRAM access pattern.
#ifndef PIC_RD_PF
#define PIC_RD_PF 0
#endif
#ifndef PIC_RD_PF_MODE      // 0: two bulk (TMA) prefetches per brick; 1: per-thread 128-B line prefetches
#define PIC_RD_PF_MODE 0
#endif

template <bool MR>
struct ReorderCap {
    static constexpr int value = MR ? PIC_RD_CAP * 13 / 14 : PIC_RD_CAP;   // MR: + the slot -> entry array
};

template <bool PUSH, bool MR>
__global__ void __launch_bounds__(kThreads, PIC_RD_MINB) k_reorder_deposit(
    Geom g, const uint32_t* __restrict__ offs, const uint32_t* __restrict__ perm, PState cur,
    const double2* __restrict__ recv, int64_t n_old, const unsigned long long* __restrict__ dcnt, PState nxt,
    double* __restrict__ rho, double* ghost, const uint32_t* __restrict__ bprev, int* __restrict__ err) {
    constexpr int CAP = ReorderCap<MR>::value;
    if (MR && dcnt) n_old = (int64_t)dcnt[DC_N];
    if (PIC_RD_PF > 0 && bprev && (PIC_RD_PF_MODE == 1 || threadIdx.x == 0)) {
        auto pf = [&](uint32_t b) {
            const uint32_t a0 = bprev[b], a1 = bprev[b + 1];
            if (a1 <= a0) return;
            if (PIC_RD_PF_MODE == 1) {       // per-thread line prefetches over the range
                const char* x0 = reinterpret_cast<const char*>(cur.xy + a0);
                const char* z0 = reinterpret_cast<const char*>(cur.zv + 2 * (int64_t)a0);
                const uint32_t nx = (16u * (a1 - a0) + 127u) / 128u, nz = (32u * (a1 - a0) + 127u) / 128u;
                for (uint32_t q = threadIdx.x; q < nx + nz; q += blockDim.x) {
                    const char* a = q < nx ? x0 + 128 * (size_t)q : z0 + 128 * (size_t)(q - nx);
                    asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(a));
                }
            } else {
                prefetch_l2_bulk(cur.xy + a0, 16u * (a1 - a0));
                prefetch_l2_bulk(cur.zv + 2 * (int64_t)a0, 32u * (a1 - a0));
            }
        };
        if (blockIdx.x < (unsigned)PIC_RD_PF) pf(blockIdx.x);
        if (blockIdx.x + (unsigned)PIC_RD_PF < gridDim.x) pf(blockIdx.x + PIC_RD_PF);
    }

    extern __shared__ double dyn_smem[];
    double2* sp0 = reinterpret_cast<double2*>(dyn_smem);               // [CAP] (x, y)
    double2* sp1 = sp0 + CAP;                                            // [CAP] (z, vz)
    double2* sp2 = sp1 + CAP;                                            // [CAP] (vx, vy)
    double* tile = reinterpret_cast<double*>(sp2 + CAP);                // [kTileSize] (16-B aligned)
    uint32_t* sperm = reinterpret_cast<uint32_t*>(tile + kTileSize);    // [CAP]
    uint32_t* soffs = sperm + CAP;                                       // [kBrick + 1]
    uint32_t* sE = soffs + kBrick + 1;                                   // [CAP] (MR): entry at slot
    uint8_t* scell = reinterpret_cast<uint8_t*>(sE + (MR ? CAP : 0));   // [CAP]
    const int t = threadIdx.x;
    const uint32_t c0 = blockIdx.x * kBrick;
    int bx, by, bz;
    unlkey(g, c0, bx, by, bz);
    soffs[t] = offs[c0 + t];
    if (t == 0) soffs[kBrick] = offs[c0 + kBrick];
    for (int q = t; q < kTileSize; q += kThreads) tile[q] = 0.0;
    __syncthreads();

    double acc[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[q] = 0.0;
    int ca = 0;
    while (ca < kBrick) {
        if (soffs[ca + 1] - soffs[ca] > (uint32_t)CAP) {
            if (t == 0) atomicExch(err, 1);
            return;
        }
        const int cb = chunk_end(soffs, ca, CAP);
        const uint32_t P0 = soffs[ca];
        const int cnt = (int)(soffs[cb] - P0);
        if ((int64_t)P0 + cnt > g.cap) {     // slab over capacity (flagged by place)
            if (t == 0) atomicExch(err + 2, 1);
            return;
        }
        for (int p = t; p < cnt; p += kThreads) sperm[p] = __ldcs(perm + P0 + p);   // read once
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
            if (MR) sE[o] = j;
            const double2* src0 = cur.xy + j;
            const double2* src1 = cur.zv + 2 * (int64_t)j;
            const double2* src2 = src1 + 1;
            if (MR && j >= n_old) {
                const double2* d = recv + 4 * ((int64_t)j - n_old);
                src0 = d; src1 = d + 1; src2 = d + 2;
            }
            cp_async16(sp0 + o, src0);
            cp_async16(sp1 + o, src1);
            cp_async16(sp2 + o, src2);
        }
        cp_async_wait_all();
        __syncthreads();
        if (MR) {   // cells holding arrivals: insertion sort by (old global key, old index)
            bool any = false;
            for (int p = s0; p < s1; ++p) any |= sE[p] >= n_old;
            if (any) {
                // the old global key of every slot once (sperm is free after the gather; the
                // old index is sE for residents, the record's high word for arrivals), then an
                // insertion sort on the cached keys: residents are already in order, arrivals
                // move past them (r02: recomputing the resident keys inside the comparison
                // loop made the last slab's reorder ~0.8 ms slower, whose arrivals from both
                // faces sort in front of the residents)
                auto rec = [&](uint32_t e) {
                    return (unsigned long long)__double_as_longlong(recv[4 * ((int64_t)e - n_old) + 3].x);
                };
                for (int p = s0; p < s1; ++p) {
                    const uint32_t e = sE[p];
                    if (e >= n_old) {
                        sperm[p] = (uint32_t)rec(e);
                    } else {
                        const double x[3] = {sp0[p].x, sp0[p].y, sp1[p].x};   // x_n (not yet drifted)
                        sperm[p] = gkey_of(g, x);
                    }
                }
                auto oldi = [&](uint32_t e) { return e >= n_old ? (uint32_t)(rec(e) >> 32) : e; };
                for (int a = s0 + 1; a < s1; ++a) {
                    const uint32_t ga = sperm[a], ea = sE[a];
                    const double2 r0 = sp0[a], r1 = sp1[a], r2 = sp2[a];
                    int b = a - 1;
                    while (b >= s0) {
                        const uint32_t gb = sperm[b];
                        if (!(ga < gb || (ga == gb && oldi(ea) < oldi(sE[b])))) break;
                        sp0[b + 1] = sp0[b]; sp1[b + 1] = sp1[b]; sp2[b + 1] = sp2[b];
                        sE[b + 1] = sE[b]; sperm[b + 1] = gb;
                        --b;
                    }
                    sp0[b + 1] = r0; sp1[b + 1] = r1; sp2[b + 1] = r2; sE[b + 1] = ea; sperm[b + 1] = ga;
                }
            }
            __syncthreads();
        }
        // drift in place (v is already kicked; arrivals arrive drifted), coalesced stores
        for (int p = t; p < cnt; p += kThreads) {
            double2 a = sp0[p], b = sp1[p];
            const double2 e = sp2[p];
            if (PUSH && !(MR && sE[p] >= n_old)) {
                double x[3] = {a.x, a.y, b.x};
                const double v[3] = {e.x, e.y, b.y};
                drift(g, x, v);
                a = make_double2(x[0], x[1]);
                b = make_double2(x[2], b.y);
                sp0[p] = a;
                sp1[p] = b;
            }
            const int64_t o = (int64_t)P0 + p;
            __stcs(nxt.xy + o, a);        // write-once: evict first, keep L2 for the gather
            st_zv_cs(nxt.zv + 2 * o, b, e);
        }
        __syncthreads();
        // CIC charge: thread per cell, its particles in stable order from shared memory
        for (int p = s0; p < s1; ++p) {
            const double x[3] = {sp0[p].x, sp0[p].y, sp1[p].x};
            cic_acc(g, x, acc);
        }
        __syncthreads();
        ca = cb;
    }
    fold_flush(g, tile, acc, t, bx, by, bz, rho, ghost);
    if (MR && bz + 4 == g.nzl && ghost != rho + (int64_t)g.nzl * g.nyr * g.rp)
        __threadfence_system();   // peer ghost atomics (PIC_P2P_GHOST=2) complete before the barrier
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
// permutation at P = 1; the step itself ranks them in shared memory only).
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

// dst += src over n doubles (n even; src may be a peer's plane: 16-B loads over NVLink)
__global__ void k_add_plane(double2* __restrict__ dst, const double2* __restrict__ src, int64_t n2) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n2) {
        const double2 a = dst[i], b = src[i];
        dst[i] = make_double2(a.x + b.x, a.y + b.y);
    }
}

// dst[r * dpitch + i] += src[r * spitch + i], i < width, r < height (pencil ghost rows)
__global__ void k_add_rows(double* __restrict__ dst, int64_t dpitch, const double* __restrict__ src,
                           int64_t spitch, int64_t width, int64_t height) {
    const int64_t tot = width * height;
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < tot; q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = q / width, i = q - r * width;
        dst[r * dpitch + i] += src[r * spitch + i];
    }
}

inline unsigned blocks(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

template <bool MR>
constexpr size_t reorder_smem() {
    constexpr int CAP = ReorderCap<MR>::value;
    return sizeof(double2) * 3 * CAP + sizeof(double) * kTileSize +
           sizeof(uint32_t) * (CAP + kBrick + 1 + (MR ? CAP : 0)) + CAP;
}

}  // namespace

cudaError_t particles_set_smem_limits() {
    cudaError_t e = cudaFuncSetAttribute(k_reorder_deposit<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)reorder_smem<false>());
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k_reorder_deposit<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)reorder_smem<false>());
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k_reorder_deposit<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)reorder_smem<true>());
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k_reorder_deposit<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)reorder_smem<true>());
    return e;
}

int reorder_cell_capacity(int nranks) { return nranks > 1 ? ReorderCap<true>::value : ReorderCap<false>::value; }

void launch_sample(const Geom& g, PState st, int64_t np, double k, double alpha, uint64_t seed,
                   cudaStream_t s) {
    if (np == 0) return;
    k_sample<<<blocks(np, kThreads), kThreads, 0, s>>>(g, st, np, k, alpha, (uint32_t)seed, (uint32_t)(seed >> 32));
}

int64_t sample_blocks(int64_t npg) { return (npg + kThreads - 1) / kThreads; }

void launch_sample_count(const Geom& g, int64_t npg, double k, double alpha, uint64_t seed,
                         uint32_t* bcount, cudaStream_t s) {
    k_sample_count<<<(unsigned)sample_blocks(npg), kThreads, 0, s>>>(g, npg, k, alpha, (uint32_t)seed,
                                                                     (uint32_t)(seed >> 32), bcount);
}

void launch_sample_write(const Geom& g, PState st, int64_t npg, double k, double alpha, uint64_t seed,
                         const uint32_t* boffs, cudaStream_t s) {
    k_sample_write<<<(unsigned)sample_blocks(npg), kThreads, 0, s>>>(g, st, npg, k, alpha, (uint32_t)seed,
                                                                     (uint32_t)(seed >> 32), boffs);
}

void launch_soa_to_pairs(const double* soa, int64_t np, PState dst, cudaStream_t s) {
    if (np == 0) return;
    k_soa_to_pairs<<<blocks(np, kThreads), kThreads, 0, s>>>(soa, np, dst);
}

void launch_pairs_to_soa(PState src, int64_t np, double* soa, cudaStream_t s) {
    if (np == 0) return;
    k_pairs_to_soa<<<blocks(np, kThreads), kThreads, 0, s>>>(src, np, soa);
}

void launch_key_import(const Geom& g, PState cur, int64_t np, uint32_t* key, uint16_t* rank,
                       uint32_t* count, int* err_flag, cudaStream_t s) {
    if (np == 0) return;
    const unsigned nb = std::min<unsigned>(blocks(np, kThreads), 148u * 32u);
    k_key_import<<<nb, kThreads, 0, s>>>(g, cur, np, key, rank, count, err_flag);
}

void launch_push_key(const Geom& g, PState cur, const uint32_t* offs, const double* E4, uint32_t* key,
                     uint16_t* rank, uint32_t* count, double2* send, uint32_t* send_count,
                     const SendSegs& segs, const PeerRecv* peers, uint32_t* bprev, int* err_flag, cudaStream_t s) {
    const unsigned nbrick = (unsigned)(((int64_t)g.n * g.nyl * g.nzl) / kBrick);
    SendBuf sb{};
    sb.data = send;
    sb.count = send_count;
    sb.segs = segs;
    // peers: the unbatched path (leavers straight into the destination from every brick)
    // only with PIC_P2P_MIG=1; by default the leavers stay local here and
    // launch_leaver_copy moves them in one stream per destination
    static const bool unbatched = [] { const char* e = getenv("PIC_P2P_MIG"); return e && e[0] == '1'; }();
    if (peers && unbatched) { sb.peers = *peers; sb.remote = 1; }
    static const bool force_mr = getenv("PIC_FORCE_MR") != nullptr;   // diagnostics
    if (PIC_RD_PF == 0 && !(PIC_PLACE_AGG && PIC_PLACE_ATOMIC)) bprev = nullptr;   // the reorder's prefetch / place_agg
    if (g.P > 1 || force_mr) k_push_key_brick<true><<<nbrick, kThreads, 0, s>>>(g, cur, offs, E4, key, rank, count, sb, bprev, err_flag);
    else k_push_key_brick<false><<<nbrick, kThreads, 0, s>>>(g, cur, offs, E4, key, rank, count, sb, bprev, err_flag);
}

bool leavers_batched() {
    const char* e = getenv("PIC_P2P_MIG");
    return !(e && e[0] == '1');
}

void launch_leaver_copy(const Geom& g, const double2* send, const SendSegs& segs, const uint32_t* send_count,
                        uint32_t* base, const PeerRecv& peers, int* err_flag, cudaStream_t s) {
    k_leaver_reserve<<<1, 32, 0, s>>>(g.P, g.rank, send_count, peers, segs, base, err_flag);
    k_leaver_copy<<<148 * 2, 256, 0, s>>>(g.P, g.rank, send, segs, send_count, base, peers);
}

void launch_key_arrivals(const Geom& g, const double2* recv, int64_t narr, int64_t n_old, uint32_t* key,
                         uint16_t* rank, uint32_t* count, int* err_flag,
                         const unsigned long long* dcnt, cudaStream_t s) {
    if (narr == 0) return;
    const unsigned nb = std::min<unsigned>(blocks(narr, kThreads), 148u * 16u);
    k_key_arrivals<<<nb, kThreads, 0, s>>>(g, recv, narr, n_old, key, rank, count, err_flag, dcnt);
}

void launch_counts_update(const Geom& g, unsigned long long* dcnt, const uint32_t* send_count,
                          int64_t np_cap, int* err_flag, cudaStream_t s) {
    k_counts_update<<<1, 1, 0, s>>>(g.P, dcnt, send_count, np_cap, err_flag);
}

void launch_set_u64(unsigned long long* p, unsigned long long v, cudaStream_t s) {
    k_set_u64<<<1, 1, 0, s>>>(p, v);
}

void launch_gkeys(const Geom& g, PState cur, int64_t np, uint32_t* key, cudaStream_t s) {
    if (np == 0) return;
    k_gkeys<<<blocks(np, kThreads), kThreads, 0, s>>>(g, cur, np, key);
}

size_t scan_scratch_bytes(int64_t n) {
    return sizeof(uint32_t) * (size_t)(blocks(n, kScanTile) + 1);
}

void launch_scan(uint32_t* count, uint32_t* offs, int64_t n, uint32_t* scratch, cudaStream_t s, bool cursor) {
    const unsigned nb = blocks(n, kScanTile);
    k_scan_reduce<<<nb, kThreads, 0, s>>>(count, n, scratch);
    k_scan_bsum<<<1, 1024, 0, s>>>(scratch, (int)nb);
    k_scan_apply<<<nb, kThreads, 0, s>>>(count, offs, n, scratch, cursor && PIC_PLACE_ATOMIC);
}

// PIC_PLACE_AGG: CTA b places the particles of brick b of the order push_key read
// ([bprev[b], bprev[b + 1])): rank within the brick's arrivals in each window cell by a
// shared atomic, one returned cursor atomic per non-empty window cell for the block base,
// then perm[base + rank] = i; particles landing outside the window take their own atomic.
__global__ void __launch_bounds__(kThreads) k_place_agg(Geom g, const uint32_t* __restrict__ key,
                                                        const uint32_t* __restrict__ bprev,
                                                        uint32_t* __restrict__ cursor, uint32_t* __restrict__ perm,
                                                        int64_t cap, int* __restrict__ err) {
    using Win = AggWin;
    __shared__ uint32_t hist[Win::NB], binkey[Win::NB], info[kInfoCap];
    const int t = threadIdx.x;
    int bx, by, bz;
    unlkey(g, blockIdx.x * kBrick, bx, by, bz);
    for (int b = t; b < Win::NB; b += kThreads) hist[b] = 0;
    const uint32_t P0 = bprev[blockIdx.x], P1 = bprev[blockIdx.x + 1];
    __syncthreads();
    for (uint32_t i = P0 + t; i < P1; i += kThreads) {
        const uint32_t k = __ldg(key + i), li = i - P0;
        int ix, iyl, izl;
        unlkey(g, k, ix, iyl, izl);
        const int b = li < (uint32_t)kInfoCap ? Win::bin(g, ix, iyl, izl, bx, by, bz) : -1;
        if (b >= 0) {
            const uint32_t lr = atomicAdd(&hist[b], 1u);
            if (lr == 0) binkey[b] = k;
            info[li] = (uint32_t)b | (lr << 12);
        } else {
            const uint32_t pos = atomicAdd(cursor + k, 1u);
            if (pos < (uint64_t)cap) perm[pos] = i;
            else atomicExch(err + 2, 1);
            if (li < (uint32_t)kInfoCap) info[li] = ~0u;
        }
    }
    __syncthreads();
    constexpr int kPer = (Win::NB + kThreads - 1) / kThreads;
    uint32_t cb[kPer], rb[kPer];
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
        const int b = t + u * kThreads;
        cb[u] = b < Win::NB ? hist[b] : 0u;
    }
#pragma unroll
    for (int u = 0; u < kPer; ++u)
        if (cb[u]) rb[u] = atomicAdd(cursor + binkey[t + u * kThreads], cb[u]);
#pragma unroll
    for (int u = 0; u < kPer; ++u)
        if (cb[u]) hist[t + u * kThreads] = rb[u];
    __syncthreads();
    const uint32_t Pe = min(P1, P0 + (uint32_t)kInfoCap);
    for (uint32_t i = P0 + t; i < Pe; i += kThreads) {
        const uint32_t v = info[i - P0];
        if (v == ~0u) continue;
        const uint32_t pos = hist[v & 0xfffu] + (v >> 12);
        if (pos < (uint64_t)cap) perm[pos] = i;
        else atomicExch(err + 2, 1);
    }
}

void launch_place(const uint32_t* key, const uint16_t* rank, int64_t np, const uint32_t* offs, uint32_t* cursor,
                  uint32_t* perm, const unsigned long long* dcnt, int64_t cap, int* err_flag, cudaStream_t s,
                  const Geom* g, const uint32_t* bprev) {
    if (np == 0) return;
    if (PIC_PLACE_AGG && PIC_PLACE_ATOMIC && g && g->P == 1 && bprev) {
        const unsigned nbrick = (unsigned)(((int64_t)g->n * g->nyl * g->nzl) / kBrick);
        k_place_agg<<<nbrick, kThreads, 0, s>>>(*g, key, bprev, cursor, perm, cap, err_flag);
        return;
    }
    k_place<<<blocks((np + 3) / 4, kThreads), kThreads, 0, s>>>(key, rank, np,
                                                                 PIC_PLACE_ATOMIC ? cursor : const_cast<uint32_t*>(offs),
                                                                 perm, dcnt, cap, err_flag);
}

void launch_reorder_deposit(const Geom& g, const uint32_t* offs, const uint32_t* perm, PState cur,
                            const double2* recv, int64_t n_old, const unsigned long long* dcnt, PState nxt,
                            int push, double* rho_buf, double* ghost, const uint32_t* bprev, int* err_flag,
                            cudaStream_t s) {
    const unsigned nbrick = (unsigned)(((int64_t)g.n * g.nyl * g.nzl) / kBrick);
    static const bool force_mr = getenv("PIC_FORCE_MR") != nullptr;   // diagnostics
    if (g.P == 1 && !force_mr) {
        if (push)
            k_reorder_deposit<true, false><<<nbrick, kThreads, reorder_smem<false>(), s>>>(g, offs, perm, cur, recv, n_old, dcnt, nxt, rho_buf, ghost, bprev, err_flag);
        else
            k_reorder_deposit<false, false><<<nbrick, kThreads, reorder_smem<false>(), s>>>(g, offs, perm, cur, recv, n_old, dcnt, nxt, rho_buf, ghost, bprev, err_flag);
    } else {
        if (push)
            k_reorder_deposit<true, true><<<nbrick, kThreads, reorder_smem<true>(), s>>>(g, offs, perm, cur, recv, n_old, dcnt, nxt, rho_buf, ghost, bprev, err_flag);
        else
            k_reorder_deposit<false, true><<<nbrick, kThreads, reorder_smem<true>(), s>>>(g, offs, perm, cur, recv, n_old, dcnt, nxt, rho_buf, ghost, bprev, err_flag);
    }
}

void launch_sort_segments(const uint32_t* offs, int64_t ncell, uint32_t* perm, cudaStream_t s) {
    k_sort_segments<<<blocks(ncell, kThreads), kThreads, 0, s>>>(offs, ncell, perm);
}

void launch_half_kick(const Geom& g, PState cur, int64_t np, const double* E4, cudaStream_t s) {
    if (np == 0) return;
    k_half_kick<<<blocks(np, kThreads), kThreads, 0, s>>>(g, cur, np, E4);
}

void launch_add_rows(double* dst, int64_t dpitch, const double* src, int64_t spitch, int64_t width, int64_t height,
                     cudaStream_t s) {
    if (width * height == 0) return;
    k_add_rows<<<std::min<unsigned>(blocks(width * height, kThreads), 148u * 8u), kThreads, 0, s>>>(
        dst, dpitch, src, spitch, width, height);
}

void launch_add_plane(double* dst, const double* src, int64_t n, cudaStream_t s) {
    k_add_plane<<<blocks(n / 2, kThreads), kThreads, 0, s>>>(reinterpret_cast<double2*>(dst),
                                                              reinterpret_cast<const double2*>(src), n / 2);
}

}  // namespace pic
