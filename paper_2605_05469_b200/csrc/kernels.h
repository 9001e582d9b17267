// kernels.h -- host-side launchers of the PIC kernels (internal to libpic.so).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "pic_device.cuh"

namespace pic {

// ------------------------------------------------------------------ FFT ----
// Spectral solve rho -> E of one z-slab (nzl planes; P = 1: the box).
// Half spectra are [.][.][px] complex rows.  Layouts of a spectral buffer (see
// SpecLayout): NORMAL [comp][z_l][y][px]; PACKED [q][comp][z_l][y_l][px] with
// y = q * nyl + y_l, nyl = n / P -- the all-to-all send/receive order of the
// transposes (P = 1: identical to NORMAL).
// REMOTE (P > 1, peer memory): the PACKED layout of the transpose's receiver --
// block q of this rank's output goes straight into rank q's buffer peer[q] at block
// `rank` (NVLink stores; no all-to-all).
struct SpecLayout {
    double2* base;
    int packed;     // 0: NORMAL, 1: PACKED, 2: REMOTE
    int ncomp;      // components in the buffer (1, 2 or 3)
    double2* const* peer;   // REMOTE: device array [P] of the receivers' buffers
};
int energy_partials(const Geom& g);
// rows of rho (nzl * n, real, pitch rp doubles) -> R2C in place
void launch_fft_x_fwd(const Geom& g, double* S0, const double2* tw, cudaStream_t s);
// y FFT of component(s) d < ncomp of src -> dst (may alias src with the same layout)
// tiles [tbeg, tend) only (default all): a tile is TW kx columns of one plane, fft_plane_tiles(n)
// tiles per plane, planes in order within each component
void launch_fft_y(const Geom& g, SpecLayout src, SpecLayout dst, int ncomp, int inverse,
                  const double2* tw, cudaStream_t s, int64_t tbeg = 0, int64_t tend = -1);
int fft_plane_tiles(int n);
int fft_zrow_tiles(int n);
// Inverse y pass of the field: src (PACKED, 2 components: phi^, E^_z after the inverse
// z pass) -> dst NORMAL 3 components: E_x = -i k_x phi, E_y = -i k_y phi, E_z.
void launch_fft_y_field(const Geom& g, SpecLayout src, SpecLayout dst, const double2* tw, cudaStream_t s);
// z pass on the ky-pencil [z][y_l][px] (all n planes of nyl ky rows): forward z FFT,
// phi^ = rho^ scale / |k|^2, 2 inverse z FFTs (phi^, E^_z = -i k_z phi^, D#6) -> out
// PACKED or REMOTE (2 components; q = z / nzl).  ky0 = rank * nyl.
void launch_fft_z_mul(const Geom& g, const double2* pencil, SpecLayout out, double scale,
                      const double2* tw, cudaStream_t s, int64_t tbeg = 0, int64_t tend = -1);   // tiles: fft_zrow_tiles(n) per ky row
// 3 components NORMAL (spec + d * nzl*n*px) -> E4 slab planes 0..nzl-1 + energy
// partials; plane 0 is also written to `halo` (the halo plane nzl of the slab below,
// on its GPU; P = 1: this slab's own), if not null.
void launch_fft_x_inv(const Geom& g, const double2* spec, double* E4, double* halo, const double2* tw,
                      double* partials, cudaStream_t s);
void launch_energy_reduce(const Geom& g, const double* partials, double* energies, cudaStream_t s);
// dst[q blk + e] = src_tab[q][rank blk + e] (complex), q < P: an all-to-all by peer pulls.
void launch_xpose_pull(double2* dst, double2* const* src_tab, int64_t blk, int rank, int P, cudaStream_t s);
// Pencils: slab field E4s [nzs + 1][n][n][4] -> y-group send blocks [Py][nzs + 1][nyl + 1][n][3] (rows
// q nyl .. q nyl + nyl, periodic), and received blocks -> the pencil field [nzl + 1][nyl + 1][n][4].
void launch_e4_pencil_pack(const double* E4s, int n, int nzs, int nyl, int Py, double* send, cudaStream_t s);
void launch_e4_pencil_unpack(const double* recv, int n, int nzs, int nyl, int Py, double* E4, cudaStream_t s);
// In-place unnormalised 3D C2C FFT of an M^3 complex grid [z][y][x], M = 2^k in [16, 1024],
// sign -1 (e^{-i k.x}) or +1; tw = W_M^m, m < M (the PIF fine grid, pif.cu).  keep > 0: the
// y / z passes only touch lines meeting the box [0, keep) u [M - keep, M) in x (and in the
// outer y of the z pass): exact for an inverse transform of a spectrum that is zero outside
// that box, and for a forward transform whose outputs outside it are not read.
// pmask (nullable): planes z with pmask[z] == 0 are neither written by the forward input nor
// read after the inverse (PIF: outside every particle tile), so the x and y passes skip them.
cudaError_t launch_fft_c2c_3d(double2* grid, int M, int sign, const double2* tw, cudaStream_t s, int keep = 0,
                              const uint32_t* pmask = nullptr);
// E4 component d <-> compact [nzl][n][n] doubles (host transfers of the field).
void launch_e4_extract(const Geom& g, const double* E4, int d, double* out, cudaStream_t s);
void launch_e4_pack(const Geom& g, const double* const comp[3], double* E4, cudaStream_t s);

// ------------------------------------------------------------- particles ----
void launch_soa_to_pairs(const double* soa, int64_t np, PState dst, cudaStream_t s);
void launch_pairs_to_soa(PState src, int64_t np, double* soa, cudaStream_t s);
// P = 1: particle j at index j; P > 1: two passes, the owned particles of all
// npg global indices written in ascending index order at boffs[block] + prefix.
void launch_sample(const Geom& g, PState st, int64_t np, double k, double alpha, uint64_t seed,
                   cudaStream_t s);
int64_t sample_blocks(int64_t npg);
void launch_sample_count(const Geom& g, int64_t npg, double k, double alpha, uint64_t seed,
                         uint32_t* bcount, cudaStream_t s);
void launch_sample_write(const Geom& g, PState st, int64_t npg, double k, double alpha, uint64_t seed,
                         const uint32_t* boffs, cudaStream_t s);
// Particles in any order: key of the current position, rank = count[key]++.
// Outside [0, L) or the slab -> err_flag[1]; a rank > 65535 -> err_flag[0].
void launch_key_import(const Geom& g, PState cur, int64_t np, uint32_t* key, uint16_t* rank,
                       uint32_t* count, int* err_flag, cudaStream_t s);
// Per-destination segments of the migration send buffer: destination r's leavers
// go to send + 4 * off[r] (64 B each), at most cap[r] of them (nranks <= 8).
struct SendSegs {
    int64_t off[8];
    int cap[8];
};
// Peer-memory migration (P > 1): leavers go straight into the destination rank's
// receive buffer peer_recv[r] (64 B records) at slots taken from its arrival counter
// peer_arr[r] (system-scope atomics over NVLink), capacity recv_cap each.
struct PeerRecv {
    double2* peer_recv[8];
    unsigned long long* peer_arr[8];
    int64_t recv_cap;
};
// Device-side particle counts of a rank (peer-memory migration): n (before the step),
// arrivals (peers add), leavers of the step, all leavers so far.
enum { DC_N = 0, DC_ARR = 1, DC_LEAVE = 2, DC_MIGRATED = 3 };
// The push of the sorted state (cell offsets offs): gather E4 through a shared tile
// per brick, kick v in place, drift; key/rank of residents.  Leavers (P > 1): with
// peers == nullptr packed into their destination's send segment (count
// send_count[dest]; full segment -> err_flag[2]); else written into the destination's
// receive buffer (full -> err_flag[2]) and counted in send_count[dest].
void launch_push_key(const Geom& g, PState cur, const uint32_t* offs, const double* E4, uint32_t* key,
                     uint16_t* rank, uint32_t* count, double2* send, uint32_t* send_count,
                     const SendSegs& segs, const PeerRecv* peers, uint32_t* bprev, int* err_flag, cudaStream_t s);
// Batched peer migration: the leavers push_key staged in this rank's send segments go
// to each destination's receive buffer at a range reserved with one system atomic on
// its arrival counter (base[P] scratch); false when PIC_P2P_MIG=1 selects the
// unbatched path inside push_key.
bool leavers_batched();
void launch_leaver_copy(const Geom& g, const double2* send, const SendSegs& segs, const uint32_t* send_count,
                        uint32_t* base, const PeerRecv& peers, int* err_flag, cudaStream_t s);
// Arrivals: key/rank at extended index n_old + a.  dcnt != null: n_old and the
// number of arrivals are read on the device (dcnt[DC_N], dcnt[DC_ARR] <= max_arr).
void launch_key_arrivals(const Geom& g, const double2* recv, int64_t narr, int64_t n_old, uint32_t* key,
                         uint16_t* rank, uint32_t* count, int* err_flag,
                         const unsigned long long* dcnt, cudaStream_t s);
// dcnt[DC_N] <- n - leavers + arrivals (> np_cap -> err_flag[2]); DC_MIGRATED += leavers;
// the arrival counter is reset for the next step.
void launch_counts_update(const Geom& g, unsigned long long* dcnt, const uint32_t* send_count,
                          int64_t np_cap, int* err_flag, cudaStream_t s);
void launch_set_u64(unsigned long long* p, unsigned long long v, cudaStream_t s);
// global Morton keys of the state (export)
void launch_gkeys(const Geom& g, PState cur, int64_t np, uint32_t* key, cudaStream_t s);
size_t scan_scratch_bytes(int64_t n);
// offs = exclusive scan of count; cursor: also leave offs in count (the place cursors)
void launch_scan(uint32_t* count, uint32_t* offs, int64_t n, uint32_t* scratch, cudaStream_t s, bool cursor = false);
// dcnt != null: the entries are dcnt[DC_N] + dcnt[DC_ARR] (<= np, read on the device).
// Sorted positions >= cap are dropped and flag err_flag[2].
void launch_place(const uint32_t* key, const uint16_t* rank, int64_t np, const uint32_t* offs, uint32_t* cursor,
                  uint32_t* perm, const unsigned long long* dcnt, int64_t cap, int* err_flag, cudaStream_t s,
                  const Geom* g = nullptr, const uint32_t* bprev = nullptr);
// Per brick: stable order inside each cell, gather through perm (entries >= n_old
// from recv; dcnt != null: n_old = dcnt[DC_N]), drift residents (push=1), store
// sorted into nxt, deposit the CIC weight sums into rho_buf planes 0..nzl-1; the
// charge of node plane nzl goes to `ghost` (plane 0 of the next slab: this buffer at
// P = 1, the peer's at P > 1 over NVLink, or this buffer's plane nzl for a separate
// fold), with system-scope atomics on the planes two GPUs share when P > 1.
void launch_reorder_deposit(const Geom& g, const uint32_t* offs, const uint32_t* perm, PState cur,
                            const double2* recv, int64_t n_old, const unsigned long long* dcnt, PState nxt,
                            int push, double* rho_buf, double* ghost, const uint32_t* bprev, int* err_flag,
                            cudaStream_t s);
void launch_sort_segments(const uint32_t* offs, int64_t ncell, uint32_t* perm, cudaStream_t s);
void launch_half_kick(const Geom& g, PState cur, int64_t np, const double* E4, cudaStream_t s);
// dst[r * dpitch + i] += src[r * spitch + i] (doubles), i < width, r < height
void launch_add_rows(double* dst, int64_t dpitch, const double* src, int64_t spitch, int64_t width, int64_t height,
                     cudaStream_t s);
void launch_add_plane(double* dst, const double* src, int64_t n, cudaStream_t s);
// -------------------------------------------------------- FD-PCG solve ----
// (pcg_kernels.cu; BJ config 5, D#26-D#31.)  Fields are
// colour-split: F[c][zl][y][x/2], c = (x + y + zl) & 1.  A PcgNbr names one field
// on this rank and on the ranks below/above (planes -1 and nzl; P = 1: own).
// Scalars sc[]: 0 sum rho, 1 (b,b), 2 (r,r), 3 (r,z), 4 previous (r,z), 5 (p,Ap).
// Every launcher ends with its one-CTA fixed-order reduction into sc (or energies).
struct PcgNbr {
    const double* own;
    const double* below;
    const double* above;
};
void launch_pcg_rho_sum(const Geom& g, const double* raw, double dscale, double* partials, double* sc,
                        cudaStream_t s);
// r = (dscale raw - sc[0]/nn) - A x -> sc[1] = (b,b), sc[2] = (r,r)
void launch_pcg_resid0(const Geom& g, const double* raw, double dscale, double* sc, double nn, PcgNbr x,
                       double* r, double* partials, cudaStream_t s);
// One red (0) / black (1) SOR half-sweep of z (in place, z.own); mode 2: z == 0 before
// (first half-sweep), 1: this colour of z == 0; dot: sc[4] = sc[3], sc[3] = (r, z).
void launch_pcg_sor(const Geom& g, int colour, int mode, bool dot, const double* r, PcgNbr z, double omega,
                    double* partials, double* sc, cudaStream_t s);
// Temporally blocked SSOR pass: ns <= pcg_tb_stages() consecutive half-sweeps
// (colour of half-sweep t = bit t-1 of seq) from zin (zero_in: z = 0, zin unused)
// into zout (!= zin); dot: sc[4] = sc[3], sc[3] = (r, zout).
int pcg_tb_stages();
void launch_pcg_ssor_pass(const Geom& g, int ns, int seq, bool zero_in, bool dot, PcgNbr r, PcgNbr zin,
                          double* zout, double omega, double* partials, double* sc, cudaStream_t s);
// pout = z + beta p (first: z), q = A pout, sc[5] = (pout, q); beta = sc[3]/sc[4].
void launch_pcg_matvec(const Geom& g, bool first, PcgNbr z, PcgNbr p, double* pout, double* q, double* sc,
                       double* partials, cudaStream_t s);
// alpha = sc[3]/sc[5]: x += alpha p, r -= alpha q, sc[2] = (r, r).
void launch_pcg_update(const Geom& g, double* x, const double* p, double* r, const double* q, double* sc,
                       double* partials, cudaStream_t s);
// E = -grad_h x -> E4 (+ plane 0 into halo if not null); energies = (W_x, W) of the slab.
void launch_pcg_gradient(const Geom& g, PcgNbr x, double* E4, double* halo, double* partials, double* energies,
                         cudaStream_t s);
void launch_pcg_unsplit(const Geom& g, const double* f, double* out, cudaStream_t s);

// ------------------------------------------------------ Q1 FEM solve ------
// (fem_kernels.cu.)  Natural [zl][y][x] fields;
// scalars sc[]: 0 sum of the load, 1 (b,b), 2 (r,r), 4 previous (r,r), 5 (p,Ap).
void launch_fem_load_sum(const Geom& g, const double* raw, double dscale, double* partials, double* sc,
                         cudaStream_t s);
void launch_fem_resid0(const Geom& g, const double* raw, double dscale, double* sc, double nn, PcgNbr x,
                       double* r, double* partials, cudaStream_t s);
void launch_fem_matvec(const Geom& g, bool first, PcgNbr r, PcgNbr p, double* pout, double* q, double* sc,
                       double* partials, cudaStream_t s);
// Split matvec (default; PIC_FEM_SPLIT=0: fused): pout = r + beta p streaming, then
// q = A pout, sc[5] = (pout, q) with the stencil on one field.
bool fem_split();
void launch_fem_paxpy(const Geom& g, const double* r, const double* p, double* pout, const double* sc,
                      cudaStream_t s);
void launch_fem_stencil(const Geom& g, PcgNbr p, double* q, double* sc, double* partials, cudaStream_t s);
void launch_fem_update(const Geom& g, double* x, const double* p, double* r, const double* q, double* sc,
                       double* partials, cudaStream_t s);
void launch_fem_gradient(const Geom& g, PcgNbr x, double* E4, double* halo, double* partials, double* energies,
                         cudaStream_t s);

// Bandwidth probes (diag_kernels.cu): returns the bytes one launch moves, < 0 for an
// unknown mode.
double launch_diag(int mode, PState cur, PState idle, const uint32_t* perm, uint32_t* scratch, int64_t np,
                   double* sink, cudaStream_t s);
cudaError_t particles_set_smem_limits();
cudaError_t fft_set_smem_limits();
// Largest cell population the reorder handles (particles staged per chunk; a larger
// cell sets the overflow flag): PIC_RD_CAP at P = 1, 13/14 of it at P > 1.
int reorder_cell_capacity(int nranks);

}  // namespace pic
