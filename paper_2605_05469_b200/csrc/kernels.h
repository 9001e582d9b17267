// kernels.h -- host-side launchers of the PIC kernels (internal to libpic.so).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "pic_device.cuh"

namespace pic {

// Six SoA particle arrays: x, y, z, vx, vy, vz.
struct PState {
    double* a[6];
};

// ------------------------------------------------------------------ FFT ----
// Spectral solve rho -> E on pitched grids:
//   rho_buf : real [n][n][rp] in (preserved).
//   E[d]    : out, real [n][n][rp]; E[0] first holds the half spectrum of rho
//             ([n][n][px] complex), then each E[d] its own half spectrum.
//   scale   : factor applied in the spectral multiply (1/N^3 times the
//             deposit's q/h^3 when rho_buf holds raw CIC weight sums).
//   tw      : twiddle table W_n^m = exp(-2 pi i m / n), m < n/2.
//   partials: >= energy_partials(g) * 3 doubles; energies: 2 doubles out
//             (W_x, W) = 1/2 h^3 sum E_x^2, 1/2 h^3 sum |E|^2.
int energy_partials(const Geom& g);
void launch_fft_x_fwd(const Geom& g, const double* rho_buf, double* spec, const double2* tw,
                      cudaStream_t s);
void launch_fft_y(const Geom& g, double* const buf[3], int ncomp, int inverse, const double2* tw,
                  cudaStream_t s);
void launch_fft_z_mul(const Geom& g, const double* rho_buf, double* const E[3], double scale,
                      const double2* tw, cudaStream_t s);
void launch_fft_x_inv(const Geom& g, double* const E[3], const double2* tw, double* partials,
                      cudaStream_t s);
void launch_energy_reduce(const Geom& g, const double* partials, double* energies, cudaStream_t s);

// ------------------------------------------------------------- particles ----
void launch_sample(const Geom& g, PState st, int64_t np, double k, double alpha, uint64_t seed,
                   cudaStream_t s);
// keys of the pushed (push=1) or current (push=0) positions; rank[i] =
// atomicAdd(count[key], 1) (arrival order in the new cell).  With push=0 a
// position outside [0, L) sets err_flag[1]; a cell with > 65535 particles err_flag[0].
void launch_push_key(const Geom& g, PState cur, int64_t np, double* const E[3], int push,
                     uint32_t* key, uint16_t* rank, uint32_t* count, int* err_flag, cudaStream_t s);
// offs[c] = sum_{c' < c} count[c'] (offs has ncell + 1 entries).
size_t scan_scratch_bytes(int64_t ncell);
void launch_scan(uint32_t* count, uint32_t* offs, int64_t ncell, uint32_t* scratch, cudaStream_t s);
// perm[offs[key[i]] + rank[i]] = i
void launch_place(const uint32_t* key, const uint16_t* rank, int64_t np, const uint32_t* offs,
                  uint32_t* perm, cudaStream_t s);
// Sort every cell's perm segment ascending in place (the stable order), for export.
void launch_sort_segments(const uint32_t* offs, int64_t ncell, uint32_t* perm, cudaStream_t s);
// Per brick of 256 cells: sort each cell's perm segment, gather (x, v)[perm],
// push (push=1), store sorted into nxt, deposit CIC weight sums into rho_buf.
void launch_reorder_deposit(const Geom& g, const uint32_t* offs, const uint32_t* perm, PState cur,
                            PState nxt, double* const E[3], int push, double* rho_buf,
                            int* err_flag, cudaStream_t s);
// Backward half kick: v <- fma(-qm_dt/2, E(x), v).
void launch_half_kick(const Geom& g, PState cur, int64_t np, double* const E[3], cudaStream_t s);
// key of every particle of the (sorted) state, for pic_get_keys_perm.
void launch_keys_only(const Geom& g, PState cur, int64_t np, uint32_t* key, cudaStream_t s);

}  // namespace pic
