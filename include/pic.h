/*
 * pic.h -- C ABI of the B200-native electrostatic PIC hot path
 * (arxiv 2605.05469, "A Comparison of Massively Parallel Performance Portable
 * Particle-in-Cell schemes ...", FFT pseudo-spectral PIC for 3D Landau damping).
 *
 * One call of pic_step() advances the PIC loop of PAPER.md Fig. 1:
 *   SOLVE   rho -> E = F^-1(-i k F(rho)/|k|^2)
 *   GATHER  E at the particles by CIC (same shape as scatter)
 *   PUSH    v += (q/m) E dt ; x += v dt ; periodic wrap
 *   SORT    stable counting sort of the particles by cell key   (BASELINE.json north_star)
 *   SCATTER CIC charge deposit of the new positions
 * for the Landau initial condition of P:140-146 in normalised units
 * (eps0 = 1, q_e = -1, m_e = 1, mean density 1), fp64 throughout.
 * "P:n" = PAPER.md line n, "S:n" = SPEC.md line n, "D#k" = DESIGN.md reading k.
 *
 * Conventions
 *  - Every function returns PIC_OK (0) or a negative pic_status.  No exception
 *    crosses the ABI and the library never prints.
 *  - Device memory: the library allocates none.  The caller (PyTorch) owns one
 *    workspace of pic_workspace_bytes() bytes on the current device and passes
 *    it to pic_init(); it must stay alive until pic_free().
 *  - Streams: every device operation is enqueued on the caller's stream
 *    (a cudaStream_t passed as void*); pic_step() is asynchronous on it, except
 *    that it copies the per-step energies to the host at the end (synchronous).
 *  - A CUDA failure poisons the context: later calls return PIC_EPOISONED.
 *  - Host buffers are plain host pointers (pageable or pinned), never retained.
 *  - Grid arrays cross the ABI as [iz][iy][ix] row-major, N^3 doubles;
 *    particle state as SoA [6][np] doubles (x, y, z, vx, vy, vz).
 */
#ifndef PIC_H
#define PIC_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct pic_ctx pic_ctx;

typedef enum {
    PIC_OK = 0,
    PIC_EINVAL = -1,       /* invalid argument (see pic_init)                      */
    PIC_ENOMEM = -2,       /* workspace too small                                  */
    PIC_ECUDA = -3,        /* a CUDA runtime call or kernel failed                 */
    PIC_ENCCL = -4,        /* an NCCL call failed (multi-GPU)                      */
    PIC_ENONFINITE = -5,   /* a field energy came out NaN/Inf                      */
    PIC_EOVERFLOW = -6,    /* particle capacity exceeded                           */
    PIC_EPOISONED = -7,    /* an earlier CUDA/NCCL error poisoned this context     */
    PIC_EUNSUPPORTED = -8, /* valid request this build does not implement          */
    PIC_ENONCONV = -9      /* PCG solver: no convergence within pcg_maxit iterations
                              (the field of the last iterate is kept; not poisoning) */
} pic_status;

/* Field solver of the PIC step.  FFT: the pseudo-spectral solve of P:171-177 (default).
 * PCG: the matrix-free finite-difference solve of P:179-181 (BJ config 5): 7-point
 * -Delta_h phi = rho - mean(rho) (periodic), conjugate gradients preconditioned by
 * red-black SSOR with pcg_inner / pcg_outer sweeps and relaxation pcg_omega,
 * warm-started from the previous step's phi, stopped at
 * ||r||_2 <= pcg_tol ||b||_2, E = -grad_h phi by central differences
 * (D#26-D#31). */
/* FEM: the matrix-free Q1 finite-element solve of P:183-195: the
 * trilinear element stiffness assembled on the fly as its 27-point stencil, lumped load
 * h^3 rho - mean, plain CG with pcg_tol / pcg_maxit, warm start, E by central
 * differences (D#33). */
typedef enum { PIC_SOLVER_FFT = 0, PIC_SOLVER_PCG = 1, PIC_SOLVER_FEM = 2 } pic_solver;

typedef struct {
    int32_t  n;         /* cells per dimension (grid N^3); power of two, 16..1024     */
    int32_t  ppc;       /* particles per cell, > 0; N_p = ppc * N^3 (Table 2)  */
    double   k;         /* perturbation wavenumber, default 0.5               */
    double   length;    /* domain length L; 0 => 2 pi / k (D#1)                */
    double   alpha;     /* perturbation amplitude, 0 <= alpha < 1; default 0.05 */
    double   dt;        /* time step > 0; default 0.05 (D#9)                   */
    uint64_t seed;      /* Philox4x32-10 key of the initial sampler (D#10)            */
    int32_t  half_kick; /* 1: v stored at half steps, backward half kick at init */
    int32_t  pgrid[2];  /* {Py, Pz} rank grid, Py Pz = nranks: {1, nranks} = z-slabs (default),
                           Py > 1 = pencils over (y, z) (BJ config 4); rank
                           r = pz Py + py owns y in [py N/Py, +N/Py), z in [pz N/Pz, +N/Pz) */
    int32_t  solver;    /* pic_solver; default PIC_SOLVER_FFT                             */
    int32_t  pcg_inner; /* PCG: SSOR inner sweeps, >= 1; default 4                */
    int32_t  pcg_outer; /* PCG: SSOR outer iterations, >= 1; default 2            */
    int32_t  pcg_maxit; /* PCG / FEM: CG iteration cap, >= 1; default 10000                */
    double   pcg_tol;   /* PCG: relative residual tolerance, > 0; default 1e-4    */
    double   pcg_omega; /* PCG: SSOR relaxation, 0 < omega < 2; default pi/2      */
    double   b_ext[3];  /* uniform external magnetic field (Eq. 1); default 0.  Nonzero:
                           the push is the Boris scheme (D#32)            */
    double   e_ext[3];  /* uniform external electric field added to E_int at the particles
                           (Eq. 1); default 0.  pic_init's half kick uses E_int only     */
} pic_params;

/* Fill *p with the Landau-damping defaults of P:146 (N=16, ppc=8, k=0.5, alpha=0.05,
 * dt=0.05, L=2 pi/k, seed=1, half_kick=1, pgrid={1,1}), solver FFT and the PCG
 * settings of P:226 / P:260 (tol 1e-4, SSOR omega = pi/2, 4 inner, 2 outer). */
pic_status pic_params_default(pic_params *p);

/* Multi-GPU (one process per GPU, nranks in {1, 2, 4, 8}): rank r = pz Py + py
 * owns the cells/nodes with z in [pz N/Pz, +N/Pz) and y in [py N/Py, +N/Py) (pgrid = {Py, Pz};
 * Py = 1: z-slabs) and the particles whose cell lies there.  The field solve always runs on
 * z-slabs of N/nranks planes (slab index = rank): pencils redistribute the charge to them and
 * the field back with one exchange in the y-group (the Py ranks sharing pz) each way, around
 * the slab FFT's own transposes.  With every workspace mapped (CUDA IPC) the
 * transposes and the y-group exchanges are copy-engine pulls of the peers' blocks, else NCCL
 * all-to-alls; pencils keep NCCL for migration, halos and ghost folds, and the FFT solver.  Rank 0 creates the NCCL id (128 bytes), the caller broadcasts it
 * (torch.distributed) and every rank passes it to pic_init. */
pic_status pic_nccl_unique_id(uint8_t id[128]);

/* The z range of a rank's domain: first plane z0, planes nz, particle capacity of the rank. */
pic_status pic_slab(const pic_params *p, int32_t rank, int32_t nranks, int32_t *z0, int32_t *nz,
                    int64_t *capacity);

/* The domain of a rank: rows [y0, y0 + ny), planes [z0, z0 + nz), particle capacity (any
 * pointer nullable).  PIC_EINVAL / PIC_EUNSUPPORTED as pic_workspace_bytes. */
pic_status pic_domain(const pic_params *p, int32_t rank, int32_t nranks, int32_t *y0, int32_t *ny, int32_t *z0,
                      int32_t *nz, int64_t *capacity);

/* Owner rank of each of np positions under the decomposition of pic_domain:
 * the rank whose domain holds the cell row i_y and plane i_z, i_d = min(floor(x_d inv_h),
 * N - 1), inv_h = (double)N / L (D#5), i.e. the rank each particle must be given to in
 * pic_set_particles.
 *   xyz   : host doubles [3][np] (x, y, z rows; xyzuvw of pic_set_particles may be passed),
 *           y and z in [0, L).
 *   owner : host int32 [np], written.
 * Pure host function (no context, no device).  PIC_EINVAL: invalid parameters (as
 * pic_workspace_bytes), NULL pointers with np > 0, or a y or z outside [0, L). */
pic_status pic_owner_ranks(const pic_params *p, int32_t nranks, const double *xyz, int64_t np,
                           int32_t *owner);

/* Bytes of device workspace pic_init needs for these parameters (rank/nranks as in
 * pic_init).  PIC_EINVAL on invalid parameters. */
pic_status pic_workspace_bytes(const pic_params *p, int32_t rank, int32_t nranks, size_t *bytes);

/* Create a context and the Landau initial state: positions by inverse
 * CDF (Newton) of (1 + alpha cos k x)/L per dimension, velocities N(0,1)^3 by
 * Box-Muller, Philox counter = particle index; particles sorted by cell key and
 * the charge deposited; optional backward half kick v <- v - (q/m) E dt/2.
 *   nccl_id   : NULL when nranks == 1; else the id from pic_nccl_unique_id on rank 0.
 *               Every rank calls every function of a context collectively (same order).
 *   workspace : device pointer, >= pic_workspace_bytes(), caller-owned.
 *   cuda_stream: cudaStream_t (void*); NULL = legacy default stream.
 * PIC_EINVAL: alpha not in [0,1), ppc <= 0, N not a power of two in [16,1024],
 *   k <= 0, dt <= 0, k L / 2 pi not a positive integer, a rank's particle index space
 *   (capacity + migration receive buffer) >= 2^32,
 *   nranks not in {1,2,4,8}, N/nranks < 4, Py Pz != nranks, pencils with N/Py < 8 or N/Pz < 4.
 * PIC_EINVAL also: solver not a pic_solver; PCG settings out of range.
 * PIC_EUNSUPPORTED: a pencil grid (Py > 1) with the PCG / FEM solver; the PCG / FEM solver
 *   at nranks > 1 without the peer-memory transport (it reads the neighbour slabs' planes
 *   over NVLink);
 * PIC_ENCCL: NCCL init failed.
 * PIC_ENOMEM: workspace_bytes too small.  PIC_ECUDA: a kernel failed. */
pic_status pic_init(const pic_params *p, int32_t rank, int32_t nranks, const uint8_t *nccl_id,
                    void *workspace, size_t workspace_bytes, void *cuda_stream, pic_ctx **out);

/* Advance nsteps PIC steps.  With the PCG solver each iteration reads the residual
 * norm on the host (one stream synchronisation per CG iteration); PIC_ENONCONV if a
 * solve does not converge.  ex_energy (nullable, nsteps doubles, host) receives
 * W_x(t_n) = 1/2 h^3 sum_nodes E_x^2 of the field solved at the start of each
 * step; t_n = n dt.  PIC_ENONFINITE if an energy is NaN/Inf. */
pic_status pic_step(pic_ctx *ctx, int32_t nsteps, double *ex_energy);

/* W_x and W = 1/2 h^3 sum |E|^2 of the latest solve (synchronises the stream). */
pic_status pic_field_energy(pic_ctx *ctx, double *ex_energy, double *total_energy);

/* Destroy the context (NULL-safe).  Never frees the caller's workspace. */
void pic_free(pic_ctx *ctx);

/* Text of the last error of ctx; NULL ctx => this thread's last pic_init error. */
const char *pic_last_error(const pic_ctx *ctx);

/* ---- host-buffer and test/bench entry points (same library, stable ABI) ---- */

/* Number of particles held by this context. */
pic_status pic_num_particles(pic_ctx *ctx, int64_t *np);

/* Particles this rank has sent to other ranks since pic_init (migration, P > 1). */
pic_status pic_migrated(pic_ctx *ctx, int64_t *migrated);

/* Transport of the P > 1 exchanges of z-slabs: *peer = 1 when every rank's workspace is
 * mapped (CUDA IPC over NVLink): halo/ghost planes and migration go through the peers'
 * buffers and the FFT transposes are copy-engine pulls; 0 for the NCCL transport
 * (all-to-all, send/recv), used when the mapping is not possible on every rank, when the
 * environment sets PIC_P2P=0 at pic_init, and for pencils (whose solve still pulls over
 * the mapping when it exists).  Always 0 at P = 1. */
pic_status pic_peer_transport(pic_ctx *ctx, int32_t *peer);

/* Copy THIS RANK's particle state to host xyzuvw[6][np] (np = pic_num_particles) in
 * canonical order (sorted by cell key, ties by the current order: at P > 1 the rank's
 * slab of the global order, SURVEY c.5).  Synchronous.  Not collective. */
pic_status pic_get_particles(pic_ctx *ctx, double *xyzuvw, int64_t np);

/* Collective (every rank of the context calls it; SURVEY §8(b) "rank 0 gathers when
 * nranks > 1"): rank 0 receives the particles of every rank in the global canonical
 * order -- a stable sort by the global Morton cell key of the rank-ordered
 * concatenation; a cell belongs to one rank, so ties keep that rank's canonical order,
 * which is the single-domain order (D#15).
 *   xyzuvw   : rank 0: host doubles [6][np_total]; other ranks: ignored (may be NULL).
 *   np_total : rank 0: the capacity of xyzuvw in particles, must equal the total;
 *              other ranks: ignored.
 *   np_out   : nullable; every rank receives the total particle count.
 * Pass xyzuvw = NULL on every rank to query the total only.  P = 1: pic_get_particles.
 * Staged through rank 0's idle particle buffer (one rank at a time, NCCL send/recv);
 * the global sort runs on rank 0's host.  PIC_EINVAL on rank 0 (and on every rank, the
 * decision is shared) if np_total differs from the total. */
pic_status pic_gather_particles(pic_ctx *ctx, double *xyzuvw, int64_t np_total, int64_t *np_out);

/* (PCG: also resets the warm start phi to 0.)
 * Replace the particle state from host xyzuvw[6][np] (P = 1: np = N_p; P > 1: this
 * rank's particles, every one inside its slab, np <= its capacity; every coordinate
 * in [0, L), else PIC_EINVAL and the offending coordinates are replaced by valid
 * ones inside the slab).  Collective at P > 1.  The state is interpreted as (x_n, v_{n-1/2})
 * (no half kick); it is sorted by cell key (stable: ties keep the given order) and
 * deposited.  With stream-ordered host copies; synchronous. */
pic_status pic_set_particles(pic_ctx *ctx, const double *xyzuvw, int64_t np);

/* Copy this rank's slab of a grid to host [nz][N][N] (P = 1: [N][N][N]): which = 0
 * -> rho (charge density of the current positions, q/h^3 scaled); 1, 2, 3 -> E_x,
 * E_y, E_z of the latest solve; 4 -> phi of the latest PCG / FEM solve (else
 * PIC_EINVAL). */
pic_status pic_get_grid(pic_ctx *ctx, int32_t which, double *host);

/* Solve for an injected charge density rho_host[nz][N][N] (this rank's slab; true
 * density, not scaled) and return E_host[3][nz][N][N] and the energies (of the
 * whole box).  Collective at P > 1.  Does not touch the
 * particles, but overwrites the context's field and charge buffers.  PCG: the
 * solve starts from phi = 0 and leaves its phi as the next step's warm start. */
pic_status pic_solve_injected(pic_ctx *ctx, const double *rho_host, double *E_host,
                              double *ex_energy, double *total_energy);

/* One gather+push+sort+deposit with an injected field E_host[3][nz][N][N] (this
 * rank's slab) instead of the solved one (the solve is skipped).  For bit-exact
 * push parity tests.  Collective at P > 1. */
pic_status pic_push_injected(pic_ctx *ctx, const double *E_host);

/* Cell keys (uint32, of the current positions in canonical order) and the
 * permutation of the latest sort (perm[i] = pre-sort index of the particle now
 * at i).  Either pointer may be NULL. */
pic_status pic_get_keys_perm(pic_ctx *ctx, uint32_t *keys, uint32_t *perm);

/* Per-stage device time (CUDA events on the context's stream), accumulated since
 * the last reset, in ms: stages[PIC_NSTAGES], launches[PIC_NSTAGES] (nullable).
 * Timing is off until pic_set_timing(ctx, 1). */
enum {
    PIC_STAGE_FFT_X_FWD = 0, PIC_STAGE_FFT_Y_FWD, PIC_STAGE_FFT_Z_MUL, PIC_STAGE_FFT_Y_INV,
    PIC_STAGE_FFT_X_INV, PIC_STAGE_ENERGY, PIC_STAGE_CLEAR, PIC_STAGE_PUSH_KEY,
    PIC_STAGE_SCAN, PIC_STAGE_PLACE, PIC_STAGE_REORDER_DEPOSIT,
    PIC_STAGE_EXCHANGE,   /* P > 1: barriers, halo/ghost planes, migration, energy sum */
    PIC_STAGE_XPOSE,      /* P > 1: the two FFT transposes (all-to-all) */
    PIC_STAGE_PCG_SSOR,   /* PCG: SSOR half-sweeps (+ barriers at P > 1) */
    PIC_STAGE_PCG_CG,     /* PCG: rhs, residual, matvec, updates, dot products, host checks */
    PIC_STAGE_PCG_FIELD,  /* PCG: central-difference gradient -> E4, energy partials */
    PIC_NSTAGES
};
pic_status pic_set_timing(pic_ctx *ctx, int32_t enable);
pic_status pic_get_timings(pic_ctx *ctx, double *ms, int64_t *launches);
pic_status pic_reset_timings(pic_ctx *ctx);
/* Name of a stage (static string) or NULL. */
const char *pic_stage_name(int32_t stage);

/* Number of kernel launches one pic_step(ctx, 1) makes (for the bench's count; PCG:
 * with the latest solve's iteration count). */
pic_status pic_launches_per_step(pic_ctx *ctx, int64_t *launches);

/* Diagnostics (not part of the step): time `reps` launches of a bandwidth
 * probe on this context's live data with the permutation of the latest sort --
 * mode 0: streaming copy of the particle state (96 B per particle), 1: the reorder's
 * gather alone through perm (100 B), 2: the place pattern alone, a 4-B scatter through
 * perm (8 B), 3: streaming read of the state (48 B).  The idle particle buffer and the
 * key array are overwritten (scratch between steps); the state is unchanged.
 * *ms = mean milliseconds per launch (CUDA events), *bytes = bytes per launch.
 * PIC_EINVAL: unknown mode or reps < 1.  Synchronous. */
pic_status pic_diag_bandwidth(pic_ctx *ctx, int32_t mode, int32_t reps, double *ms, double *bytes);

/* PCG / FEM (CG) solver statistics: iterations of the latest solve (-1: not converged), total
 * iterations and solves since pic_init, relative residual ||r||/||b|| of the latest
 * solve.  Any pointer may be NULL.  PIC_EINVAL for an FFT context. */
pic_status pic_pcg_stats(pic_ctx *ctx, int32_t *last_iters, int64_t *total_iters, int64_t *solves,
                         double *last_relres);

#ifdef __cplusplus
}
#endif
#endif /* PIC_H */
