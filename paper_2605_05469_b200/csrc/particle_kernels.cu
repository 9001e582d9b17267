// particle_kernels.cu -- particle side of the PIC step on sm_100a.
//
// One step (after the solve) is four kernels over HBM-resident SoA fp64 state:
//   push_key : stream x, v in sorted order, gather E (CIC), push, key of the new
//              cell, count[key] += 1.  Nothing but the 4-byte key is written.
//   scan     : offs = exclusive scan of count (3 kernels, 4096-cell tiles).
//   place    : perm[atomicAdd(cursor[key[i]], 1)] = i.
//   reorder_deposit : one CTA per Morton brick of 256 cells (8 x 8 x 4).  Sorts
//              each cell's perm segment ascending (= the stable order), gathers
//              x, v through perm, recomputes the identical push, streams x', v'
//              sorted into the other buffer, and deposits the new charge: each
//              thread owns one cell and sums its particles' 8 corner weights in
//              registers, the brick combines them into a 9 x 9 x 5 node tile in
//              shared memory in eight conflict-free passes, and the tile is
//              flushed with one fp64 global reduction per node.
// The push is computed twice (push_key, reorder_deposit) from bit-identical code
// (pic_device.cuh) instead of writing x', v' twice: 48 B/particle less traffic.
#include <algorithm>

#include "kernels.h"

namespace pic {

namespace {

constexpr int kThreads = 256;
constexpr int kBrick = 256;     // cells per reorder/deposit CTA (Morton 8 bits)
constexpr int kCap = 4096;      // particles staged per chunk

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
    for (int d = 0; d < 3; ++d) {
        const double target = u[d] * g.L;
        double x = target;
        for (int it = 0; it < 32; ++it) {
            const double F = __dsub_rn(__dadd_rn(x, __dmul_rn(ak, sin(k * x))), target);
            const double dF = __dadd_rn(1.0, __dmul_rn(alpha, cos(k * x)));
            const double dx = __ddiv_rn(F, dF);
            x = __dsub_rn(x, dx);
            if (fabs(dx) < 1e-12) break;
        }
        st.a[d][j] = wrap(x, g.L);
    }
    const double two_pi = 6.283185307179586476925286766559;
    const double r1 = sqrt(-2.0 * log(1.0 - u[3]));
    const double r2 = sqrt(-2.0 * log(1.0 - u[5]));
    st.a[3][j] = r1 * cos(two_pi * u[4]);
    st.a[4][j] = r1 * sin(two_pi * u[4]);
    st.a[5][j] = r2 * cos(two_pi * u[6]);
}

// ----------------------------------------------------------- push + key ----
// Grid-stride over the sorted particles with the next particle's x, v loads in
// flight while the current one gathers E.  rank[i] = the particle's arrival
// order in its new cell (return value of the count atomic), so the placement
// needs no second atomic.
template <bool PUSH>
__global__ void __launch_bounds__(kThreads) k_push_key(Geom g, PState cur, int64_t np,
                                                       const double* __restrict__ Ex,
                                                       const double* __restrict__ Ey,
                                                       const double* __restrict__ Ez,
                                                       uint32_t* __restrict__ key,
                                                       uint16_t* __restrict__ rank,
                                                       uint32_t* __restrict__ count,
                                                       int* __restrict__ err) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    double xn[3], vn[3];
    if (i < np) {
#pragma unroll
        for (int d = 0; d < 3; ++d) { xn[d] = __ldg(cur.a[d] + i); vn[d] = __ldg(cur.a[3 + d] + i); }
    }
    for (; i < np; i += stride) {
        double x[3] = {xn[0], xn[1], xn[2]}, v[3] = {vn[0], vn[1], vn[2]};
        const int64_t inext = i + stride;
        if (inext < np) {
#pragma unroll
            for (int d = 0; d < 3; ++d) { xn[d] = __ldg(cur.a[d] + inext); vn[d] = __ldg(cur.a[3 + d] + inext); }
        }
        if (PUSH) {
            gather_push(g, Ex, Ey, Ez, x, v);
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

__global__ void __launch_bounds__(kThreads) k_keys_only(Geom g, PState cur, int64_t np,
                                                        uint32_t* __restrict__ key) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= np) return;
    double x[3] = {cur.a[0][i], cur.a[1][i], cur.a[2][i]};
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
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= np) return;
    perm[__ldg(offs + __ldg(key + i)) + __ldg(rank + i)] = (uint32_t)i;
}

// ------------------------------------------------- reorder + push + deposit -
// One CTA per Morton brick of 256 cells (8 x 8 x 4).  Phases per chunk of the
// brick's sorted positions:
//   1. stage perm[chunk] in shared memory; one thread per cell insertion-sorts
//      its segment ascending (= the stable order, D#14);
//   2. one thread per sorted position p (a warp covers 32 consecutive p):
//      gather x, v through perm (next particle prefetched), push, store x', v'
//      at p, compute its 8 CIC corner weights, and reduce them over the lanes of
//      the same cell (segmented shuffle scan; positions are cell-sorted); the
//      head lane of each cell segment adds the 8 sums to that cell's
//      accumulator in shared memory;
//   3. after the last chunk, the 256 cell accumulators are folded into the
//      9 x 9 x 5 node tile in eight conflict-free passes and the tile is flushed
//      with one fp64 global reduction (RED.ADD.F64) per node.
template <bool PUSH>
__global__ void __launch_bounds__(kThreads, 3) k_reorder_deposit(
    Geom g, const uint32_t* __restrict__ offs, const uint32_t* __restrict__ perm, PState cur,
    PState nxt, const double* __restrict__ Ex, const double* __restrict__ Ey,
    const double* __restrict__ Ez, double* __restrict__ rho, int* __restrict__ err) {
    __shared__ uint32_t soffs[kBrick + 1];
    __shared__ uint32_t sperm[kCap];
    __shared__ double sacc[8][kBrick];
    __shared__ double tile[9 * 9 * 5];
    const int t = threadIdx.x, lane = t & 31;
    const uint32_t c0 = blockIdx.x * kBrick;
    int bx, by, bz;
    unmorton(c0, bx, by, bz);
    soffs[t] = offs[c0 + t];
    if (t == 0) soffs[kBrick] = offs[c0 + kBrick];
#pragma unroll
    for (int q = 0; q < 8; ++q) sacc[q][t] = 0.0;
    for (int q = t; q < 9 * 9 * 5; q += kThreads) tile[q] = 0.0;
    __syncthreads();

    int ca = 0;
    while (ca < kBrick) {
        // largest cb with soffs[cb] - soffs[ca] <= kCap (uniform across the CTA)
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
        for (int p = t; p < cnt; p += kThreads) sperm[p] = __ldg(perm + P0 + p);
        __syncthreads();
        if (t >= ca && t < cb) {  // insertion sort of this cell's segment: stable order
            const int s0 = (int)(soffs[t] - P0), s1 = (int)(soffs[t + 1] - P0);
            for (int a = s0 + 1; a < s1; ++a) {
                const uint32_t vv = sperm[a];
                int b = a - 1;
                while (b >= s0 && sperm[b] > vv) { sperm[b + 1] = sperm[b]; --b; }
                sperm[b + 1] = vv;
            }
        }
        __syncthreads();

        const int nit = (cnt + kThreads - 1) / kThreads;
        int p = t;
        double xn[3], vn[3];
        bool okn = p < cnt;
        if (okn) {
            const uint32_t j = sperm[p];
#pragma unroll
            for (int d = 0; d < 3; ++d) { xn[d] = __ldg(cur.a[d] + j); vn[d] = __ldg(cur.a[3 + d] + j); }
        }
        for (int it = 0; it < nit; ++it, p += kThreads) {
            double x[3] = {xn[0], xn[1], xn[2]}, v[3] = {vn[0], vn[1], vn[2]};
            const bool ok = okn;
            okn = p + kThreads < cnt;
            if (okn) {   // prefetch the next particle of this thread
                const uint32_t j = sperm[p + kThreads];
#pragma unroll
                for (int d = 0; d < 3; ++d) { xn[d] = __ldg(cur.a[d] + j); vn[d] = __ldg(cur.a[3 + d] + j); }
            }
            double w8[8];
            int lc = 1024 + lane;   // unique sentinel for idle lanes
            if (ok) {
                if (PUSH) gather_push(g, Ex, Ey, Ez, x, v);
                const int64_t o = (int64_t)P0 + p;
#pragma unroll
                for (int d = 0; d < 3; ++d) {
                    nxt.a[d][o] = x[d];
                    nxt.a[3 + d][o] = v[d];
                }
                int ii[3];
                double w[3][2];
                cic_weights(g, x, ii, w);
#pragma unroll
                for (int q = 0; q < 8; ++q)
                    w8[q] = __dmul_rn(__dmul_rn(w[0][q & 1], w[1][(q >> 1) & 1]), w[2][q >> 2]);
                lc = (int)morton(ii[0] - bx, ii[1] - by, ii[2] - bz);
            } else {
#pragma unroll
                for (int q = 0; q < 8; ++q) w8[q] = 0.0;
            }
            // segmented suffix sums over lanes of equal cell (cell-sorted positions)
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int olc = __shfl_down_sync(0xffffffffu, lc, o);
                const bool same = lane + o < 32 && olc == lc;
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const double ov = __shfl_down_sync(0xffffffffu, w8[q], o);
                    if (same) w8[q] += ov;
                }
            }
            const int plc = __shfl_up_sync(0xffffffffu, lc, 1);
            if (ok && (lane == 0 || plc != lc)) {
#pragma unroll
                for (int q = 0; q < 8; ++q) atomicAdd(&sacc[q][lc], w8[q]);
            }
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
        tile[((lz + c) * 9 + (ly + b)) * 9 + (lx + a)] += sacc[q][t];
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
                                                        const double* __restrict__ Ex,
                                                        const double* __restrict__ Ey,
                                                        const double* __restrict__ Ez) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= np) return;
    double x[3] = {cur.a[0][i], cur.a[1][i], cur.a[2][i]};
    double ep[3];
    gather_E(g, Ex, Ey, Ez, x, ep);
    const double hk = -0.5 * g.qm_dt;   // v_{-1/2} = v_0 - (q/m) E dt/2
#pragma unroll
    for (int d = 0; d < 3; ++d) cur.a[3 + d][i] = __fma_rn(hk, ep[d], cur.a[3 + d][i]);
}

// perm segments of every cell sorted ascending in place (export of the stable
// permutation; the step itself sorts them in shared memory only).
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

}  // namespace

void launch_sample(const Geom& g, PState st, int64_t np, double k, double alpha, uint64_t seed,
                   cudaStream_t s) {
    if (np == 0) return;
    k_sample<<<blocks(np, kThreads), kThreads, 0, s>>>(g, st, np, k, alpha, (uint32_t)seed,
                                                        (uint32_t)(seed >> 32));
}

void launch_push_key(const Geom& g, PState cur, int64_t np, double* const E[3], int push,
                     uint32_t* key, uint16_t* rank, uint32_t* count, int* err_flag, cudaStream_t s) {
    if (np == 0) return;
    const unsigned nb = std::min<unsigned>(blocks(np, kThreads), 148u * 32u);
    if (push)
        k_push_key<true><<<nb, kThreads, 0, s>>>(g, cur, np, E[0], E[1], E[2], key, rank, count, err_flag);
    else
        k_push_key<false><<<nb, kThreads, 0, s>>>(g, cur, np, E[0], E[1], E[2], key, rank, count, err_flag);
}

void launch_keys_only(const Geom& g, PState cur, int64_t np, uint32_t* key, cudaStream_t s) {
    if (np == 0) return;
    k_keys_only<<<blocks(np, kThreads), kThreads, 0, s>>>(g, cur, np, key);
}

size_t scan_scratch_bytes(int64_t ncell) {
    return sizeof(uint32_t) * (size_t)(blocks(ncell, kScanTile) + 1);
}

void launch_scan(uint32_t* count, uint32_t* offs, int64_t ncell, uint32_t* scratch, cudaStream_t s) {
    const unsigned nb = blocks(ncell, kScanTile);
    k_scan_reduce<<<nb, kThreads, 0, s>>>(count, ncell, scratch);
    k_scan_bsum<<<1, 1024, 0, s>>>(scratch, (int)nb);
    k_scan_apply<<<nb, kThreads, 0, s>>>(count, offs, ncell, scratch);
}

void launch_place(const uint32_t* key, const uint16_t* rank, int64_t np, const uint32_t* offs,
                  uint32_t* perm, cudaStream_t s) {
    if (np == 0) return;
    k_place<<<blocks(np, kThreads), kThreads, 0, s>>>(key, rank, np, offs, perm);
}

void launch_reorder_deposit(const Geom& g, const uint32_t* offs, const uint32_t* perm, PState cur,
                            PState nxt, double* const E[3], int push, double* rho_buf,
                            int* err_flag, cudaStream_t s) {
    const unsigned nbrick = (unsigned)(((int64_t)g.n * g.n * g.n) / kBrick);
    if (push)
        k_reorder_deposit<true><<<nbrick, kThreads, 0, s>>>(g, offs, perm, cur, nxt, E[0], E[1], E[2],
                                                             rho_buf, err_flag);
    else
        k_reorder_deposit<false><<<nbrick, kThreads, 0, s>>>(g, offs, perm, cur, nxt, E[0], E[1], E[2],
                                                              rho_buf, err_flag);
}

void launch_sort_segments(const uint32_t* offs, int64_t ncell, uint32_t* perm, cudaStream_t s) {
    k_sort_segments<<<blocks(ncell, kThreads), kThreads, 0, s>>>(offs, ncell, perm);
}

void launch_half_kick(const Geom& g, PState cur, int64_t np, double* const E[3], cudaStream_t s) {
    if (np == 0) return;
    k_half_kick<<<blocks(np, kThreads), kThreads, 0, s>>>(g, cur, np, E[0], E[1], E[2]);
}

}  // namespace pic
