// kernels.h -- host-side launchers of the PIC kernels (internal to libpic.so).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "pic_device.cuh"

namespace pic {

// ------------------------------------------------------------------ FFT ----
// Spectral solve rho -> E on pitched grids [n][n][rp] (real) /
// [n][n][px] (complex half spectra):
//   S0     : in: rho (raw CIC weight sums); R2C x and y in place; after the z pass
//            it holds E^_z and after the inverse y pass its y-inverse.
//   S1, S2 : out of the z pass: E^_x, E^_y (then their y-inverses).
//   E4     : out: node records (E_x, E_y, E_z, 0), [n][n][n][4].
//   scale  : factor of the spectral multiply (q/h^3 / N^3 for raw weight sums).
//   tw     : twiddle table W_n^m = exp(-2 pi i m / n), m < n.
//   partials: 3 * energy_partials(g) doubles; energies: 2 doubles out
//            (W_x, W) = 1/2 h^3 sum E_x^2, 1/2 h^3 sum |E|^2.
int energy_partials(const Geom& g);
void launch_fft_x_fwd(const Geom& g, double* S0, const double2* tw, cudaStream_t s);
void launch_fft_y(const Geom& g, double* const buf[3], int ncomp, int inverse, const double2* tw,
                  cudaStream_t s);
void launch_fft_z_mul(const Geom& g, double* S0, double* S1, double* S2, double scale,
                      const double2* tw, cudaStream_t s);
void launch_fft_x_inv(const Geom& g, const double* const spec[3], double* E4, const double2* tw,
                      double* partials, cudaStream_t s);
void launch_energy_reduce(const Geom& g, const double* partials, double* energies, cudaStream_t s);
// E4 component d <-> compact [n^3] doubles (host transfers of the field).
void launch_e4_extract(const Geom& g, const double* E4, int d, double* out, cudaStream_t s);
void launch_e4_pack(const Geom& g, const double* const comp[3], double* E4, cudaStream_t s);

// ------------------------------------------------------------- particles ----
// Host layout [6][np] (x, y, z, vx, vy, vz) <-> device pairs (pic_device.cuh).
void launch_soa_to_pairs(const double* soa, int64_t np, PState dst, cudaStream_t s);
void launch_pairs_to_soa(PState src, int64_t np, double* soa, cudaStream_t s);
void launch_sample(const Geom& g, PState st, int64_t np, double k, double alpha, uint64_t seed,
                   cudaStream_t s);
// keys of the pushed (push=1: particles sorted by cell with offsets offs; gather
// E4 through a shared-memory tile per brick, kick v in place, drift) or current
// (push=0, any order) positions; rank[i] = atomicAdd(count[key], 1).  With push=0
// a position outside [0, L) sets err_flag[1]; a rank > 65535 sets err_flag[0].
void launch_push_key(const Geom& g, PState cur, int64_t np, const uint32_t* offs, const double* E4,
                     int push, uint32_t* key, uint16_t* rank, uint32_t* count, int* err_flag,
                     cudaStream_t s);
// offs[c] = sum_{c' < c} count[c'] (offs has ncell + 1 entries).
size_t scan_scratch_bytes(int64_t ncell);
void launch_scan(const uint32_t* count, uint32_t* offs, int64_t ncell, uint32_t* scratch,
                 cudaStream_t s);
// perm[offs[key[i]] + rank[i]] = i
void launch_place(const uint32_t* key, const uint16_t* rank, int64_t np, const uint32_t* offs,
                  uint32_t* perm, cudaStream_t s);
// Per brick of 256 cells: stable order inside each cell, gather (x, v) through
// perm, drift (push=1), store sorted into nxt, deposit CIC weight sums into S0.
void launch_reorder_deposit(const Geom& g, const uint32_t* offs, const uint32_t* perm, PState cur,
                            PState nxt, int push, double* rho_buf, int* err_flag, cudaStream_t s);
// Backward half kick: v <- fma(-qm_dt/2, E(x), v).
void launch_half_kick(const Geom& g, PState cur, int64_t np, const double* E4, cudaStream_t s);
// key of every particle of the (sorted) state, for pic_get_keys_perm.
void launch_keys_only(const Geom& g, PState cur, int64_t np, uint32_t* key, cudaStream_t s);
// Sort every cell's perm segment ascending in place (the stable order), for export.
void launch_sort_segments(const uint32_t* offs, int64_t ncell, uint32_t* perm, cudaStream_t s);

}  // namespace pic
