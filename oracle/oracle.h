/*
 * oracle.h -- plain, slow, obviously-correct CPU oracle of the electrostatic
 * PIC step (3D Landau damping, FFT pseudo-spectral Poisson solve, CIC, leapfrog).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load this library.
 * The product path (paper_2605_05469_b200/) never imports, links or executes
 * anything under oracle/, and this file shares no code, header, table or
 * constant generator with the CUDA path.
 *
 * Citation key: "P:n" = PAPER.md line n, "S:n" = SPEC.md line n,
 * "D#k" = reading k in DESIGN.md section "Readings of the paper".
 *
 * Conventions (all fp64):
 *   grid arrays      : [iz][iy][ix] row-major, index (iz*N + iy)*N + ix, N^3 doubles.
 *   vector fields    : E[d][N^3], d = 0 (x), 1 (y), 2 (z).
 *   particle state   : xv[6][np] structure of arrays: x, y, z, vx, vy, vz.
 *   units            : eps0 = 1, q_e = -1, m_e = 1, mean density 1,
 *                      so macro charge q = -L^3/np and q/m = -1 (D#2).
 */
#ifndef PIC_ORACLE_H
#define PIC_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Thread count of every oracle function (SURVEY c.5): 1 (default) = serial,
 * bitwise-reproducible parity mode; T > 1 = OpenMP-deterministic mode -- results
 * identical to serial except the summation order of the deposit (two-colour
 * z-slabs) and of the field energy (T fixed chunks), deterministic for a fixed T. */
void oracle_set_threads(int32_t threads);
int32_t oracle_get_threads(void);

/* Philox4x32-10 counter-based RNG (D#10); out = philox(ctr, key). */
void oracle_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
/* The 8 uniforms u_0..u_7 in [0,1) of particle j (D#10). */
void oracle_uniforms(uint64_t seed, uint64_t j, double u[8]);
/* Landau initial condition: x_d ~ (1+alpha cos(k x))/L by inverse CDF
 * (Newton), v ~ N(0,1)^3 by Box-Muller.  Writes xv[6][np] in index order j. */
void oracle_sample_landau(int64_t np, double k, double L, double alpha, uint64_t seed,
                          double *xv);

/* Cell index along one dim: floor(x*inv_h) clamped to N-1 (D#5). */
int32_t oracle_cell_index(double x, double inv_h, int32_t n);
/* Cell key: Morton (bit-interleaved) order of (ix, iy, iz), x fastest (D#14). */
uint32_t oracle_morton_key(int32_t ix, int32_t iy, int32_t iz, int32_t n);
/* keys[j] of every particle from its current position. */
void oracle_keys(int32_t n, double L, int64_t np, const double *xv, uint32_t *keys);
/* Stable sort of the particles by cell key (D#14); perm[i] = old index of the
 * particle now at i; xv is permuted in place. */
void oracle_sort(int32_t n, double L, int64_t np, double *xv, uint32_t *perm);

/* CIC deposit, P:105 / S:132-140: rho[node] = q/h^3 * sum_j w(node, x_j). */
void oracle_deposit(int32_t n, double L, int64_t np, const double *xv, double q, double *rho);
/* Pseudo-spectral solve: E = F^-1(-i k F(rho)/|k|^2), zero mode and
 * the d-th Nyquist plane removed from E_d (D#6).  radix-2 FFT along each axis on
 * the full complex array.  Returns max |imag| of the inverse transforms. */
double oracle_solve_fft(int32_t n, double L, const double *rho, double *E);
/* The same solve by brute-force direct DFT (O(N^6)); N <= 16 only. */
double oracle_solve_dft(int32_t n, double L, const double *rho, double *E);
/* Field energy, P:231 / S:72-80: wx = 1/2 h^3 sum E_x^2, w = 1/2 h^3 sum |E|^2. */
void oracle_field_energy(int32_t n, double L, const double *E, double *wx, double *w);
/* CIC gather, P:105 / S:141-149: Ep[d][j] = sum_corners w * E_d(node). */
void oracle_gather(int32_t n, double L, int64_t np, const double *xv, const double *E,
                   double *Ep);
/* Leapfrog kick-drift + periodic wrap, P:106-109 / S:150-167:
 * v <- v + (q/m) dt E_p ; x <- x + v dt ; wrap into [0, L). */
void oracle_push(double L, int64_t np, double *xv, const double *Ep, double qm_dt, double dt);
/* Periodic wrap of one coordinate. */
double oracle_wrap(double x, double L);

/* Whole PIC loop (Fig. 1).  State (x_n, v_{n-1/2}) in xv, any order.
 * The particles are first put in canonical order (stable sort by key); then
 * nsteps x {scatter -> solve (+energy) -> gather -> push -> wrap -> sort}.
 * ex_energy / tot_energy (nullable) receive W_x(t_n), W(t_n) for each step.
 * perm_last (nullable, np entries) receives the last step's sort permutation. */
void oracle_run(int32_t n, double L, double dt, int64_t np, double *xv, int32_t nsteps,
                double *ex_energy, double *tot_energy, uint32_t *perm_last);
/* Backward half kick: v <- v - (q/m) E(x_0) dt/2, x unchanged. */
void oracle_half_kick(int32_t n, double L, double dt, int64_t np, double *xv);

/* ---- FD-PCG Poisson solve (BJ config 5; D#26-D#31) ---- */
/* y = -Delta_h x, 7-point second-order stencil, periodic. */
void oracle_laplacian_fd(int32_t n, double L, const double *x, double *y);
/* z = M^-1 r: red-black SSOR, `outer` x (`inner` x red+black, `inner` x black+red)
 * SOR half-sweeps with relaxation omega from z = 0 (D#28). */
void oracle_ssor(int32_t n, double L, const double *r, double *z, double omega, int32_t inner,
                 int32_t outer);
/* Preconditioned CG for -Delta_h x = b from the guess in x (warm start); precond
 * 1 = SSOR, 0 = none; stop at ||r||^2 <= tol^2 ||b||^2.  Returns iterations or -1. */
int32_t oracle_pcg(int32_t n, double L, const double *b, double *x, double tol, int32_t precond,
                   double omega, int32_t inner, int32_t outer, int32_t maxit, double *relres);
/* E_d = (phi(m - e_d) - phi(m + e_d)) inv_h / 2 (D#30). */
void oracle_gradient_central(int32_t n, double L, const double *phi, double *E);
/* b = rho - mean(rho); PCG warm-started from phi; E = -grad_h phi. */
int32_t oracle_solve_pcg(int32_t n, double L, const double *rho, double *phi, double *E, double tol,
                         double omega, int32_t inner, int32_t outer, int32_t maxit, double *relres);
/* oracle_run with the PCG solve; phi in/out (warm start); iters (nullable) per step. */
void oracle_run_pcg(int32_t n, double L, double dt, int64_t np, double *xv, int32_t nsteps,
                    double *ex_energy, double *tot_energy, double *phi, double tol, double omega,
                    int32_t inner, int32_t outer, int32_t maxit, int32_t *iters);
void oracle_half_kick_pcg(int32_t n, double L, double dt, int64_t np, double *xv, double *phi, double tol,
                          double omega, int32_t inner, int32_t outer, int32_t maxit);

/* ---- external fields and the Boris push (Eq. 1, 3-4: P:97; D#32) ---- */
/* t = (q/m)(dt/2) B_ext, s = 2 t / (1 + |t|^2). */
void oracle_boris_coeffs(double dt, const double *b_ext, double t[3], double s[3]);
/* Kick (leapfrog if B_ext = 0, else Boris) with E = E_p + E_ext, drift, wrap. */
void oracle_push_ext(double L, int64_t np, double *xv, const double *Ep, double dt, const double *b_ext,
                     const double *e_ext);
/* oracle_run (FFT solve) with uniform external fields B_ext, E_ext. */
void oracle_run_ext(int32_t n, double L, double dt, int64_t np, double *xv, int32_t nsteps,
                    double *ex_energy, double *tot_energy, const double *b_ext, const double *e_ext);

/* ---- matrix-free Q1 FEM solve (D#33) ---- */
void oracle_fem_element_stiffness(double h, double Ae[64]);
void oracle_fem_apply(int32_t n, double L, const double *x, double *y);
int32_t oracle_fem_cg(int32_t n, double L, const double *b, double *x, double tol, int32_t maxit,
                      double *relres);
int32_t oracle_solve_fem(int32_t n, double L, const double *rho, double *phi, double *E, double tol,
                         int32_t maxit, double *relres);
void oracle_run_fem(int32_t n, double L, double dt, int64_t np, double *xv, int32_t nsteps,
                    double *ex_energy, double *tot_energy, double *phi, double tol, int32_t maxit,
                    int32_t *iters);
void oracle_half_kick_fem(int32_t n, double L, double dt, int64_t np, double *xv, double *phi, double tol,
                          int32_t maxit);

#ifdef __cplusplus
}
#endif
#endif
