/*
 * pif.h -- C ABI of the Particle-in-Fourier field solve and its NUFFTs
 * (arxiv 2605.05469 section "Particle-in-Fourier (PIF)", and Appendix A,
 * P:423-467).  Exported by libpic.so next to pic.h.
 * "P:n" = PAPER.md line n, "S:n" = SPEC.md line n, "D#k" = DESIGN.md reading k.
 *
 * Conventions (as pic.h: PIC_OK or a negative pic_status, no exceptions, no prints):
 *  - Modes: K_N = (2 pi / L) [-N/2, N/2 - 1]^3, N a power of two, 8 <= N <= 512 (the fine
 *    grid M = 2N is transformed by the repo's own FFT passes, M <= 1024).  A mode
 *    array is N^3 complex values (interleaved re, im doubles) indexed
 *    [(nz + N/2) N + (ny + N/2)] N + (nx + N/2) (n ascending).
 *  - Positions: device SoA x[3][np] doubles (x, y, z), each in [0, L).  Weights f[np],
 *    charges q[np]: device doubles.  Outputs are device buffers owned by the caller.
 *  - Accuracy eps (1e-4): window of w = ceil(log10(1/eps)) + 2 fine-grid points
 *    per dimension, the "exponential of semicircle" exp(beta (sqrt(1 - z^2) - 1)),
 *    beta = 2.30 w, on the sigma = 2 oversampled grid M = 2N (D#34).
 *  - Device memory: the library allocates none; the caller owns one workspace of
 *    pic_pif_workspace_bytes() bytes (fine grid M^3 complex, two N^3 complex spectra, the
 *    FFT's twiddle table) and the stream; both must outlive the plan.
 *  - The uniform FFT on the fine grid is this library's radix-8 Stockham passes (in-place
 *    C2C, one pass per axis; the passes of the FFT-PIC solve), like
 *    the spreading, interpolation, mode selection, deconvolution and Poisson step.
 *  - A CUDA failure poisons the plan: later calls return PIC_EPOISONED.
 */
#ifndef PIC_PIF_H
#define PIC_PIF_H
#include "pic.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct pic_pif pic_pif;

/* Workspace bytes for modes N, domain length L, accuracy eps and up to np_max particles per
 * call (pure host function).
 * np_max > 0 reserves the binned path (4 B per particle + 12 B per bin of 8^3 fine cells, and
 * a second M^3 complex fine grid so the PIF solve gathers E_x, E_y, E_z in one pass;
 * PIC_PIF_SPLIT_INTERP=1 keeps two passes): particles counting-sorted into bins, spreading
 * and interpolation through shared-memory tiles; it applies
 * when 2N is a multiple of 8 and w <= 8 (eps >= 1e-6) and np <= np_max (else, or with
 * PIC_PIF_BINNED=0 in the environment, one global atomic per window point).  PIC_EINVAL: N
 * not a power of two in [8, 512], L <= 0, eps outside [1e-14, 1), np_max outside [0, 2^32). */
pic_status pic_pif_workspace_bytes(int32_t n, double length, double eps, int64_t np_max, size_t *bytes);

/* Create a plan on the current device over `workspace` (>= pic_pif_workspace_bytes) and
 * `stream` (cudaStream_t as void*; NULL = legacy default).  Computes the deconvolution
 * table 1 / psi^(n) on the device.  PIC_ENOMEM: workspace too small. */
pic_status pic_pif_create(int32_t n, double length, double eps, int64_t np_max, void *workspace,
                          size_t bytes, void *stream, pic_pif **out);

/* Type-1 NUFFT, Eq. (p2f) / (type1nufft): fhat(k) = sum_j f_j e^{-i k.x_j}
 * for k in K_N, computed as D chi F C f.  fhat: device [N^3][2] doubles.  Asynchronous. */
pic_status pic_nufft_type1(pic_pif *p, int64_t np, const double *x, const double *f, double *fhat);

/* Type-2 NUFFT, Eq. (f2p) / (type2nufft): out_j = sum_k fhat(k) e^{+i k.x_j},
 * computed as C^T F^-1 chi^T D fhat.  out: device [np][2] doubles.  Asynchronous. */
pic_status pic_nufft_type2(pic_pif *p, int64_t np, const double *x, const double *fhat, double *out);

/* PIF field solve: rho^ = type-1 of the charges q; phi^ = rho^ / |k|^2 (D#8, k = 0
 * removed, D#3); E^ = -i k phi^ with the unpaired -N/2 planes dropped (D#36);
 * E(x_j) = L^-3 type-2(E^)(x_j) (D#35).  E: device [3][np] doubles.  energy (host, 3
 * doubles, nullable): W_d = 1/(2 L^3) sum_k |E^_d|^2 (D#37); if non-null the call
 * synchronises the stream.  PIC_ENONFINITE if an energy is NaN/Inf. */
pic_status pic_pif_solve(pic_pif *p, int64_t np, const double *x, const double *q, double *E,
                         double *energy);

/* PIF time loop (Fig. 1, with the PIF solve in place of deposit + solve + gather):
 * nsteps x { E = pic_pif_solve(x); W_x(t_n) -> ex_energy[n] (D#12); v += qm dt E;
 * x += v dt; wrap into [0, L) (D#9, the PIC push) }.  x, v: device [3][np] (updated in
 * place); q: device [np]; E: device [3][np] scratch (holds the last step's field).
 * ex_energy: host [nsteps] or NULL (one synchronisation at the end).  PIC_EINVAL: nsteps
 * outside [1, 4096]. */
pic_status pic_pif_step(pic_pif *p, int64_t np, double *x, double *v, const double *q, double *E,
                        double qm, double dt, int32_t nsteps, double *ex_energy);

/* Per-stage device time (CUDA events on the plan's stream) accumulated over the calls since
 * timing was enabled, ms[PIC_PIF_NSTAGES]; launches[PIC_PIF_NSTAGES] nullable.  Enabling
 * timing makes every call synchronise at its end. */
enum {
    PIC_PIF_SPREAD = 0, /* C: clear + spread the weights onto the fine grid          */
    PIC_PIF_FFT,        /* F / F^-1 on the M^3 fine grid (own C2C passes)             */
    PIC_PIF_MODES,      /* chi, D, Poisson, -i k, energy partials (type 1 side)       */
    PIC_PIF_FILL,       /* chi^T D: the fine grid from the spectrum (type 2 side)     */
    PIC_PIF_INTERP,     /* C^T: the window sums at the particles                      */
    PIC_PIF_PUSH,       /* pic_pif_step: kick, drift, wrap                             */
    PIC_PIF_BIN,        /* binned path: counting sort of the particles into bins       */
    PIC_PIF_NSTAGES
};
/* Decomposed PIF over nranks processes (one GPU each; collective: every rank calls it once
 * after pic_pif_create, with the NCCL id rank 0 made by pic_nccl_unique_id): each rank holds
 * its own particles; from then on pic_nufft_type1 and the PIF solve (pic_pif_solve,
 * pic_pif_step) sum the selected modes over the ranks (ncclAllReduce of N^3 complex) before
 * the Poisson step, so every rank has the field of all the particles, the energies are
 * global, and each rank's type-2 gather serves its own particles (the paper's PIF
 * parallelisation: the particle sums are distributed, the modes reduced).
 * Every rank calls every later function of the plan collectively.  nranks == 1: no-op.
 * PIC_EINVAL: bad rank / nranks, NULL id, or already attached.  PIC_ENCCL: init failed. */
pic_status pic_pif_attach_nccl(pic_pif *p, int32_t rank, int32_t nranks, const uint8_t nccl_id[128]);

pic_status pic_pif_set_timing(pic_pif *p, int32_t enable);
pic_status pic_pif_get_timings(pic_pif *p, double *ms, int64_t *launches);

/* Window width w of the plan (fine-grid points per dimension) and fine size M. */
pic_status pic_pif_window(pic_pif *p, int32_t *w, int32_t *m);

/* Last error message of the plan (or of the last failed create, p = NULL). */
const char *pic_pif_last_error(const pic_pif *p);

/* Free the host-side plan (the caller frees the workspace). */
void pic_pif_free(pic_pif *p);

#ifdef __cplusplus
}
#endif
#endif /* PIC_PIF_H */
