// diag_kernels.cu -- bandwidth probes on a context's live particle data (diagnostics
// for DESIGN.md §6, not part of the step): what the access patterns of the sort's
// kernels can reach on this device, with the real permutation of the latest step.
//   mode 0: streaming copy of the state, cur -> idle buffer (48 B read + 48 B written)
//   mode 1: the reorder's gather alone: idle[o] = cur[perm[o]] (4 + 48 B read, 48 B written)
//   mode 2: the place pattern alone: scratch[perm[o]] = o (4 B read, 4 B scattered write)
//   mode 3: streaming read of the state (48 B read)
#include "kernels.h"

namespace pic {
namespace {

__global__ void __launch_bounds__(256) k_diag_copy(PState src, PState dst, int64_t np) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < np; i += (int64_t)gridDim.x * blockDim.x) {
        double2 b, c;
        const double2 a = __ldcs(src.xy + i);
        ld_zv(src.zv + 2 * i, b, c);
        __stcs(dst.xy + i, a);
        st_zv_cs(dst.zv + 2 * i, b, c);
    }
}

__global__ void __launch_bounds__(256) k_diag_gather(PState src, PState dst, const uint32_t* __restrict__ perm,
                                                     int64_t np) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < np; o += 2 * stride) {
        const int64_t o2 = o + stride;
        const uint32_t j = __ldcs(perm + o);
        const uint32_t j2 = o2 < np ? __ldcs(perm + o2) : 0u;
        double2 b, c, b2, c2;
        const double2 a = __ldg(src.xy + j);
        ld_zv(src.zv + 2 * (int64_t)j, b, c);
        const double2 a2 = __ldg(src.xy + j2);
        ld_zv(src.zv + 2 * (int64_t)j2, b2, c2);
        __stcs(dst.xy + o, a);
        st_zv_cs(dst.zv + 2 * o, b, c);
        if (o2 < np) {
            __stcs(dst.xy + o2, a2);
            st_zv_cs(dst.zv + 2 * o2, b2, c2);
        }
    }
}

__global__ void __launch_bounds__(256) k_diag_scatter(const uint32_t* __restrict__ perm, uint32_t* __restrict__ out,
                                                      int64_t np) {
    for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < np; o += (int64_t)gridDim.x * blockDim.x)
        out[__ldcs(perm + o)] = (uint32_t)o;
}

__global__ void __launch_bounds__(256) k_diag_read(PState src, int64_t np, double* sink) {
    double s = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < np; i += (int64_t)gridDim.x * blockDim.x) {
        double2 b, c;
        const double2 a = __ldcs(src.xy + i);
        ld_zv(src.zv + 2 * i, b, c);
        s += a.x + a.y + b.x + b.y + c.x + c.y;
    }
    if (s == 12345.678) *sink = s;   // keeps the loads
}

}  // namespace

double launch_diag(int mode, PState cur, PState idle, const uint32_t* perm, uint32_t* scratch, int64_t np,
                   double* sink, cudaStream_t s) {
    const unsigned grid = 148 * 8;
    switch (mode) {
    case 0: k_diag_copy<<<grid, 256, 0, s>>>(cur, idle, np); return 96.0 * np;
    case 1: k_diag_gather<<<grid, 256, 0, s>>>(cur, idle, perm, np); return 100.0 * np;
    case 2: k_diag_scatter<<<grid, 256, 0, s>>>(perm, scratch, np); return 8.0 * np;
    case 3: k_diag_read<<<grid, 256, 0, s>>>(cur, np, sink); return 48.0 * np;
    default: return -1.0;
    }
}

}  // namespace pic
