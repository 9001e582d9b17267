/*
 * oracle.c -- plain CPU oracle of the electrostatic PIC step.  TEST
 * INFRASTRUCTURE ONLY (see oracle.h): never used by the product path.
 *
 * Build: gcc -O2 -ffp-contract=off -fPIC -shared (fma() only where written).
 * Every function follows the paper's definition in the paper's order; no
 * blocking, fusion or reordering.  Citations: P:n = PAPER.md line n,
 * S:n = SPEC.md line n, D#k = DESIGN.md reading k.
 */
#include "oracle.h"

#include <complex.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------ threads ---- *
 * SURVEY c.1 "Implementation of the oracle" / c.5 "Oracle modes": threads = 1 is
 * the serial, bitwise-reproducible parity mode; threads > 1 is the
 * OpenMP-deterministic mode (fixed thread count, static schedules, a stable
 * two-level sort that equals the serial one, a two-colour z-slab deposit and
 * fixed-order reductions).  Only the deposit's and the energy's summation order
 * depend on the thread count; every other stage computes bit-identical results
 * (the same per-particle / per-line arithmetic). */
static int g_threads = 1;

void oracle_set_threads(int32_t t) { g_threads = t < 1 ? 1 : t; }
int32_t oracle_get_threads(void) { return g_threads; }

/* ------------------------------------------------------------------ RNG ---- */
/* Philox4x32-10 (Salmon et al., Random123), D#10. */
static void mulhilo32(uint32_t a, uint32_t b, uint32_t *hi, uint32_t *lo) {
    uint64_t p = (uint64_t)a * (uint64_t)b;
    *hi = (uint32_t)(p >> 32);
    *lo = (uint32_t)p;
}

void oracle_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
    const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
    const uint32_t W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
    uint32_t c[4] = {ctr_in[0], ctr_in[1], ctr_in[2], ctr_in[3]};
    uint32_t k[2] = {key_in[0], key_in[1]};
    for (int r = 0; r < 10; ++r) {
        if (r > 0) { k[0] += W0; k[1] += W1; }
        uint32_t hi0, lo0, hi1, lo1;
        mulhilo32(M0, c[0], &hi0, &lo0);
        mulhilo32(M1, c[2], &hi1, &lo1);
        uint32_t n0 = hi1 ^ c[1] ^ k[0];
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c[3] ^ k[1];
        uint32_t n3 = lo0;
        c[0] = n0; c[1] = n1; c[2] = n2; c[3] = n3;
    }
    out[0] = c[0]; out[1] = c[1]; out[2] = c[2]; out[3] = c[3];
}

/* u_t = (w_t >> 11) * 2^-53, w_{2b} = r0 | r1<<32, w_{2b+1} = r2 | r3<<32 with
 * (r0..r3) = philox((j lo, j hi, b, 0), (seed lo, seed hi)), b = 0..3 (D#10). */
void oracle_uniforms(uint64_t seed, uint64_t j, double u[8]) {
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    for (uint32_t b = 0; b < 4; ++b) {
        uint32_t ctr[4] = {(uint32_t)j, (uint32_t)(j >> 32), b, 0u};
        uint32_t r[4];
        oracle_philox4x32_10(ctr, key, r);
        uint64_t w0 = (uint64_t)r[0] | ((uint64_t)r[1] << 32);
        uint64_t w1 = (uint64_t)r[2] | ((uint64_t)r[3] << 32);
        u[2 * b] = (double)(w0 >> 11) * 0x1p-53;
        u[2 * b + 1] = (double)(w1 >> 11) * 0x1p-53;
    }
}

double oracle_wrap(double x, double L) {
    /* wrap into [0, L); x = L maps to 0. */
    if (x >= L) {
        x = x - L;
    } else if (x < 0.0) {
        x = x + L;
        if (x >= L) x = 0.0;
    }
    return x;
}

/* Inverse CDF of the 1D marginal (1 + alpha cos(k x))/L, P:143-146:
 * F(x) = x + (alpha/k) sin(k x) - u L = 0, Newton from x = u L, |dx| < 1e-12 or
 * 32 iterations. */
static double landau_position(double u, double k, double L, double alpha) {
    double target = u * L;
    double x = target;
    for (int it = 0; it < 32; ++it) {
        double F = x + (alpha / k) * sin(k * x) - target;
        double dF = 1.0 + alpha * cos(k * x);
        double dx = F / dF;
        x = x - dx;
        if (fabs(dx) < 1e-12) break;
    }
    return oracle_wrap(x, L);
}

void oracle_sample_landau(int64_t np, double k, double L, double alpha, uint64_t seed,
                          double *xv) {
    const double two_pi = 6.283185307179586476925286766559;
#pragma omp parallel for schedule(static) num_threads(g_threads)
    for (int64_t j = 0; j < np; ++j) {
        double u[8];
        oracle_uniforms(seed, (uint64_t)j, u);
        for (int d = 0; d < 3; ++d) xv[d * np + j] = landau_position(u[d], k, L, alpha);
        /* Box-Muller: (vx, vy) from (u3, u4), vz from (u5, u6). */
        double r1 = sqrt(-2.0 * log(1.0 - u[3]));
        double r2 = sqrt(-2.0 * log(1.0 - u[5]));
        xv[3 * np + j] = r1 * cos(two_pi * u[4]);
        xv[4 * np + j] = r1 * sin(two_pi * u[4]);
        xv[5 * np + j] = r2 * cos(two_pi * u[6]);
    }
}

/* ------------------------------------------------------------ keys/sort ---- */
int32_t oracle_cell_index(double x, double inv_h, int32_t n) {
    int32_t i = (int32_t)floor(x * inv_h);
    if (i >= n) i = n - 1;  /* x just below L rounding up (D#5) */
    if (i < 0) i = 0;
    return i;
}

uint32_t oracle_morton_key(int32_t ix, int32_t iy, int32_t iz, int32_t n) {
    uint32_t key = 0;
    for (int b = 0; (1 << b) < n; ++b) {
        key |= (uint32_t)((ix >> b) & 1) << (3 * b);
        key |= (uint32_t)((iy >> b) & 1) << (3 * b + 1);
        key |= (uint32_t)((iz >> b) & 1) << (3 * b + 2);
    }
    return key;
}

void oracle_keys(int32_t n, double L, int64_t np, const double *xv, uint32_t *keys) {
    const double inv_h = (double)n / L;
#pragma omp parallel for schedule(static) num_threads(g_threads)
    for (int64_t j = 0; j < np; ++j) {
        int32_t ix = oracle_cell_index(xv[0 * np + j], inv_h, n);
        int32_t iy = oracle_cell_index(xv[1 * np + j], inv_h, n);
        int32_t iz = oracle_cell_index(xv[2 * np + j], inv_h, n);
        keys[j] = oracle_morton_key(ix, iy, iz, n);
    }
}

/* OpenMP-deterministic stable sort (threads > 1): a stable partition of the
 * particle indices into T contiguous key ranges (per-chunk histograms, fixed
 * chunk order), then a stable counting sort of each range by key.  Both steps
 * keep index order among equal keys, so perm equals the serial counting sort's. */
static void sort_perm_parallel(int64_t np, const uint32_t *keys, int64_t ncell, uint32_t *perm, int T) {
    int64_t *hist = (int64_t *)calloc((size_t)T * T, sizeof(int64_t));   /* [chunk][range] */
    uint32_t *part = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)(np > 0 ? np : 1));
    int64_t *rstart = (int64_t *)calloc((size_t)T + 1, sizeof(int64_t));
#pragma omp parallel for schedule(static, 1) num_threads(T)
    for (int c = 0; c < T; ++c) {
        const int64_t j0 = np * c / T, j1 = np * (c + 1) / T;
        for (int64_t j = j0; j < j1; ++j) hist[(int64_t)c * T + (int64_t)keys[j] * T / ncell] += 1;
    }
    int64_t run = 0;
    for (int b = 0; b < T; ++b) {         /* range-major, chunk-minor: stable */
        rstart[b] = run;
        for (int c = 0; c < T; ++c) {
            const int64_t v = hist[(int64_t)c * T + b];
            hist[(int64_t)c * T + b] = run;
            run += v;
        }
    }
    rstart[T] = run;
#pragma omp parallel for schedule(static, 1) num_threads(T)
    for (int c = 0; c < T; ++c) {
        const int64_t j0 = np * c / T, j1 = np * (c + 1) / T;
        for (int64_t j = j0; j < j1; ++j) part[hist[(int64_t)c * T + (int64_t)keys[j] * T / ncell]++] = (uint32_t)j;
    }
#pragma omp parallel for schedule(static, 1) num_threads(T)
    for (int b = 0; b < T; ++b) {
        const int64_t k0 = (b * ncell + T - 1) / T, k1 = ((b + 1) * ncell + T - 1) / T;   /* keys of range b */
        int64_t *start = (int64_t *)calloc((size_t)(k1 - k0) + 1, sizeof(int64_t));
        for (int64_t i = rstart[b]; i < rstart[b + 1]; ++i) start[keys[part[i]] - k0 + 1] += 1;
        for (int64_t k = 0; k < k1 - k0; ++k) start[k + 1] += start[k];
        for (int64_t i = rstart[b]; i < rstart[b + 1]; ++i) perm[rstart[b] + start[keys[part[i]] - k0]++] = part[i];
        free(start);
    }
    free(rstart);
    free(part);
    free(hist);
}

void oracle_sort(int32_t n, double L, int64_t np, double *xv, uint32_t *perm) {
    /* Stable counting sort by cell key: ties keep the current order (D#14). */
    const int64_t ncell = (int64_t)n * n * n;
    const int T = g_threads;
    uint32_t *keys = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)(np > 0 ? np : 1));
    double *tmp = (double *)malloc(sizeof(double) * (size_t)(np > 0 ? np : 1));
    oracle_keys(n, L, np, xv, keys);
    if (T == 1) {
        int64_t *start = (int64_t *)calloc((size_t)ncell + 1, sizeof(int64_t));
        for (int64_t j = 0; j < np; ++j) start[keys[j] + 1] += 1;
        for (int64_t c = 0; c < ncell; ++c) start[c + 1] += start[c];
        for (int64_t j = 0; j < np; ++j) perm[start[keys[j]]++] = (uint32_t)j;
        free(start);
    } else {
        sort_perm_parallel(np, keys, ncell, perm, T);
    }
    for (int a = 0; a < 6; ++a) {
        double *col = xv + (int64_t)a * np;
#pragma omp parallel for schedule(static) num_threads(T)
        for (int64_t i = 0; i < np; ++i) tmp[i] = col[perm[i]];
#pragma omp parallel for schedule(static) num_threads(T)
        for (int64_t i = 0; i < np; ++i) col[i] = tmp[i];
    }
    free(tmp);
    free(keys);
}

/* ------------------------------------------------------------ scatter ----- */
static int64_t node(int32_t n, int32_t ix, int32_t iy, int32_t iz) {
    return ((int64_t)((iz % n + n) % n) * n + ((iy % n + n) % n)) * n + ((ix % n + n) % n);
}

/* The eight CIC corner weights of particle j added to rho. */
static void deposit_one(int32_t n, double inv_h, int64_t np, const double *xv, int64_t j, double *rho) {
    int32_t i[3];
    double w[3][2];
    for (int d = 0; d < 3; ++d) {
        double s = xv[d * np + j] * inv_h;
        i[d] = oracle_cell_index(xv[d * np + j], inv_h, n);
        double f = s - (double)i[d];
        w[d][0] = 1.0 - f;
        w[d][1] = f;
    }
    for (int c = 0; c < 2; ++c)
        for (int b = 0; b < 2; ++b)
            for (int a = 0; a < 2; ++a) {
                double wt = (w[0][a] * w[1][b]) * w[2][c];
                rho[node(n, i[0] + a, i[1] + b, i[2] + c)] += wt;
            }
}

/* OpenMP-deterministic deposit (threads > 1, SURVEY c.5): S (even, <= n) z-slabs of
 * cell planes; slab s = the particles whose cell plane iz has iz S / n = s, kept in
 * index order by a stable partition.  A slab touches its own node planes and the
 * next one, so slabs of one colour (s mod 2) never share a node: colour 0, then
 * colour 1, each slab summed in index order.  Deterministic for a fixed S. */
static void deposit_slabs(int32_t n, double inv_h, int64_t np, const double *xv, double *rho, int T) {
    int S = 2 * T;
    if (S > n) S = n;
    int64_t *hist = (int64_t *)calloc((size_t)T * S, sizeof(int64_t));   /* [chunk][slab] */
    int64_t *sstart = (int64_t *)calloc((size_t)S + 1, sizeof(int64_t));
    uint32_t *idx = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)(np > 0 ? np : 1));
#pragma omp parallel for schedule(static, 1) num_threads(T)
    for (int c = 0; c < T; ++c)
        for (int64_t j = np * c / T; j < np * (c + 1) / T; ++j)
            hist[(int64_t)c * S + (int64_t)oracle_cell_index(xv[2 * np + j], inv_h, n) * S / n] += 1;
    int64_t run = 0;
    for (int s = 0; s < S; ++s) {
        sstart[s] = run;
        for (int c = 0; c < T; ++c) {
            const int64_t v = hist[(int64_t)c * S + s];
            hist[(int64_t)c * S + s] = run;
            run += v;
        }
    }
    sstart[S] = run;
#pragma omp parallel for schedule(static, 1) num_threads(T)
    for (int c = 0; c < T; ++c)
        for (int64_t j = np * c / T; j < np * (c + 1) / T; ++j)
            idx[hist[(int64_t)c * S + (int64_t)oracle_cell_index(xv[2 * np + j], inv_h, n) * S / n]++] = (uint32_t)j;
    for (int colour = 0; colour < 2; ++colour) {
#pragma omp parallel for schedule(static, 1) num_threads(T)
        for (int s = colour; s < S; s += 2)
            for (int64_t i = sstart[s]; i < sstart[s + 1]; ++i) deposit_one(n, inv_h, np, xv, idx[i], rho);
    }
    free(idx);
    free(sstart);
    free(hist);
}

void oracle_deposit(int32_t n, double L, int64_t np, const double *xv, double q, double *rho) {
    const double inv_h = (double)n / L;
    const int64_t nn = (int64_t)n * n * n;
    for (int64_t m = 0; m < nn; ++m) rho[m] = 0.0;
    if (g_threads == 1) {
        for (int64_t j = 0; j < np; ++j) deposit_one(n, inv_h, np, xv, j, rho);
    } else {
        deposit_slabs(n, inv_h, np, xv, rho, g_threads);
    }
    const double scale = q * ((inv_h * inv_h) * inv_h);
#pragma omp parallel for schedule(static) num_threads(g_threads)
    for (int64_t m = 0; m < nn; ++m) rho[m] = scale * rho[m];
}

/* -------------------------------------------------------------- solve ----- */
/* In-place radix-2 complex FFT of one strided line, sign = -1 forward
 * (e^{-i k x}), +1 inverse (unnormalised).  Twiddles cos/sin(2 pi j / N). */
static void fft_line(double complex *a, int32_t n, int64_t stride, int sign) {
    const double two_pi = 6.283185307179586476925286766559;
    for (int32_t i = 1, j = 0; i < n; ++i) {
        int32_t bit = n >> 1;
        for (; j & bit; bit >>= 1) j ^= bit;
        j ^= bit;
        if (i < j) {
            double complex t = a[i * stride];
            a[i * stride] = a[j * stride];
            a[j * stride] = t;
        }
    }
    for (int32_t len = 2; len <= n; len <<= 1) {
        for (int32_t i = 0; i < n; i += len) {
            for (int32_t m = 0; m < len / 2; ++m) {
                double ang = sign * two_pi * (double)m / (double)len;
                double complex w = cos(ang) + I * sin(ang);
                double complex u = a[(i + m) * stride];
                double complex v = a[(i + m + len / 2) * stride] * w;
                a[(i + m) * stride] = u + v;
                a[(i + m + len / 2) * stride] = u - v;
            }
        }
    }
}

static void fft3d(double complex *c, int32_t n, int sign) {
    /* every line is transformed by the same code whatever the thread count */
#pragma omp parallel for schedule(static) num_threads(g_threads)
    for (int32_t iz = 0; iz < n; ++iz)          /* along x */
        for (int32_t iy = 0; iy < n; ++iy) fft_line(c + ((int64_t)iz * n + iy) * n, n, 1, sign);
#pragma omp parallel for schedule(static) num_threads(g_threads)
    for (int32_t iz = 0; iz < n; ++iz)          /* along y */
        for (int32_t ix = 0; ix < n; ++ix) fft_line(c + (int64_t)iz * n * n + ix, n, n, sign);
#pragma omp parallel for schedule(static) num_threads(g_threads)
    for (int32_t iy = 0; iy < n; ++iy)          /* along z */
        for (int32_t ix = 0; ix < n; ++ix) fft_line(c + (int64_t)iy * n + ix, n, (int64_t)n * n, sign);
}

/* Mode number n_d in [-N/2, N/2-1] of array index idx. */
static int32_t mode_of(int32_t idx, int32_t n) { return idx < n / 2 ? idx : idx - n; }

/* Spectral field of mode (ix,iy,iz): E_d = -i k_d rho / |k|^2, with E = 0 at
 * n = 0 and E_d = 0 where n_d = -N/2 (D#6). P:175. */
static void spectral_field(int32_t n, double L, int32_t ix, int32_t iy, int32_t iz,
                           double complex rhohat, double complex Ehat[3]) {
    const double two_pi = 6.283185307179586476925286766559;
    int32_t idx[3] = {ix, iy, iz};
    double kv[3];
    double k2 = 0.0;
    for (int d = 0; d < 3; ++d) {
        kv[d] = two_pi * (double)mode_of(idx[d], n) / L;
        k2 += kv[d] * kv[d];
    }
    for (int d = 0; d < 3; ++d) {
        if (k2 == 0.0 || idx[d] == n / 2) Ehat[d] = 0.0;
        else Ehat[d] = -I * kv[d] * rhohat / k2;
    }
}

double oracle_solve_fft(int32_t n, double L, const double *rho, double *E) {
    const int64_t nn = (int64_t)n * n * n;
    double complex *rh = (double complex *)malloc(sizeof(double complex) * (size_t)nn);
    double complex *eh = (double complex *)malloc(sizeof(double complex) * (size_t)nn * 3);
#pragma omp parallel for schedule(static) num_threads(g_threads)
    for (int64_t m = 0; m < nn; ++m) rh[m] = rho[m];
    fft3d(rh, n, -1);
#pragma omp parallel for schedule(static) num_threads(g_threads)
    for (int32_t iz = 0; iz < n; ++iz)
        for (int32_t iy = 0; iy < n; ++iy)
            for (int32_t ix = 0; ix < n; ++ix) {
                int64_t m = ((int64_t)iz * n + iy) * n + ix;
                double complex e3[3];
                spectral_field(n, L, ix, iy, iz, rh[m], e3);
                for (int d = 0; d < 3; ++d) eh[d * nn + m] = e3[d];
            }
    double max_imag = 0.0;
    for (int d = 0; d < 3; ++d) {
        fft3d(eh + d * nn, n, +1);
#pragma omp parallel for schedule(static) num_threads(g_threads) reduction(max : max_imag)
        for (int64_t m = 0; m < nn; ++m) {
            double complex v = eh[d * nn + m] / (double)nn;
            E[d * nn + m] = creal(v);
            if (fabs(cimag(v)) > max_imag) max_imag = fabs(cimag(v));
        }
    }
    free(eh);
    free(rh);
    return max_imag;
}

double oracle_solve_dft(int32_t n, double L, const double *rho, double *E) {
    /* rhohat(n) = sum_m rho(m) e^{-2 pi i n.m/N};  E_d(m) = N^-3 sum_n Ehat_d(n) e^{+2 pi i n.m/N}. */
    const double two_pi = 6.283185307179586476925286766559;
    const int64_t nn = (int64_t)n * n * n;
    double complex *eh = (double complex *)malloc(sizeof(double complex) * (size_t)nn * 3);
    for (int64_t kk = 0; kk < nn; ++kk) {
        int32_t kx = (int32_t)(kk % n), ky = (int32_t)((kk / n) % n), kz = (int32_t)(kk / ((int64_t)n * n));
        double complex acc = 0.0;
        for (int64_t m = 0; m < nn; ++m) {
            int32_t mx = (int32_t)(m % n), my = (int32_t)((m / n) % n), mz = (int32_t)(m / ((int64_t)n * n));
            int64_t ph = ((int64_t)kx * mx + (int64_t)ky * my + (int64_t)kz * mz) % n;
            double ang = -two_pi * (double)ph / (double)n;
            acc += rho[m] * (cos(ang) + I * sin(ang));
        }
        double complex e3[3];
        spectral_field(n, L, kx, ky, kz, acc, e3);
        for (int d = 0; d < 3; ++d) eh[d * nn + kk] = e3[d];
    }
    double max_imag = 0.0;
    for (int d = 0; d < 3; ++d) {
        for (int64_t m = 0; m < nn; ++m) {
            int32_t mx = (int32_t)(m % n), my = (int32_t)((m / n) % n), mz = (int32_t)(m / ((int64_t)n * n));
            double complex acc = 0.0;
            for (int64_t kk = 0; kk < nn; ++kk) {
                int32_t kx = (int32_t)(kk % n), ky = (int32_t)((kk / n) % n), kz = (int32_t)(kk / ((int64_t)n * n));
                int64_t ph = ((int64_t)kx * mx + (int64_t)ky * my + (int64_t)kz * mz) % n;
                double ang = two_pi * (double)ph / (double)n;
                acc += eh[d * nn + kk] * (cos(ang) + I * sin(ang));
            }
            acc = acc / (double)nn;
            E[d * nn + m] = creal(acc);
            if (fabs(cimag(acc)) > max_imag) max_imag = fabs(cimag(acc));
        }
    }
    free(eh);
    return max_imag;
}

void oracle_field_energy(int32_t n, double L, const double *E, double *wx, double *w) {
    const int64_t nn = (int64_t)n * n * n;
    const double h = L / (double)n;
    const double h3 = (h * h) * h;
    double sx = 0.0, s = 0.0;
    if (g_threads == 1) {
        for (int64_t m = 0; m < nn; ++m) {
            double ex = E[m], ey = E[nn + m], ez = E[2 * nn + m];
            sx += ex * ex;
            s += ex * ex + ey * ey + ez * ez;
        }
    } else {          /* fixed-order reduction: T sequential chunk sums, added in chunk order */
        const int T = g_threads;
        double *px = (double *)calloc((size_t)T, sizeof(double)), *ps = (double *)calloc((size_t)T, sizeof(double));
#pragma omp parallel for schedule(static, 1) num_threads(T)
        for (int c = 0; c < T; ++c)
            for (int64_t m = nn * c / T; m < nn * (c + 1) / T; ++m) {
                double ex = E[m], ey = E[nn + m], ez = E[2 * nn + m];
                px[c] += ex * ex;
                ps[c] += ex * ex + ey * ey + ez * ez;
            }
        for (int c = 0; c < T; ++c) { sx += px[c]; s += ps[c]; }
        free(px);
        free(ps);
    }
    *wx = 0.5 * h3 * sx;
    *w = 0.5 * h3 * s;
}

/* --------------------------------------------------------- gather/push ---- */
void oracle_gather(int32_t n, double L, int64_t np, const double *xv, const double *E,
                   double *Ep) {
    const double inv_h = (double)n / L;
    const int64_t nn = (int64_t)n * n * n;
#pragma omp parallel for schedule(static) num_threads(g_threads)
    for (int64_t j = 0; j < np; ++j) {
        int32_t i[3];
        double w[3][2];
        for (int d = 0; d < 3; ++d) {
            double s = xv[d * np + j] * inv_h;
            i[d] = oracle_cell_index(xv[d * np + j], inv_h, n);
            double f = s - (double)i[d];
            w[d][0] = 1.0 - f;
            w[d][1] = f;
        }
        double acc[3] = {0.0, 0.0, 0.0};
        for (int c = 0; c < 2; ++c)
            for (int b = 0; b < 2; ++b)
                for (int a = 0; a < 2; ++a) {
                    double wt = (w[0][a] * w[1][b]) * w[2][c];
                    int64_t m = node(n, i[0] + a, i[1] + b, i[2] + c);
                    for (int d = 0; d < 3; ++d) acc[d] = fma(wt, E[d * nn + m], acc[d]);
                }
        for (int d = 0; d < 3; ++d) Ep[d * np + j] = acc[d];
    }
}

void oracle_push(double L, int64_t np, double *xv, const double *Ep, double qm_dt, double dt) {
#pragma omp parallel for schedule(static) num_threads(g_threads)
    for (int64_t j = 0; j < np; ++j) {
        for (int d = 0; d < 3; ++d) {
            double v = fma(qm_dt, Ep[d * np + j], xv[(3 + d) * np + j]);   /* kick */
            double x = fma(v, dt, xv[d * np + j]);                        /* drift */
            xv[(3 + d) * np + j] = v;
            xv[d * np + j] = oracle_wrap(x, L);
        }
    }
}

/* ------------------------------------------------------------ PIC loop ---- */
void oracle_half_kick(int32_t n, double L, double dt, int64_t np, double *xv) {
    const int64_t nn = (int64_t)n * n * n;
    const double q = -((L * L) * L) / (double)np;
    const double qm = -1.0;
    double *rho = (double *)malloc(sizeof(double) * (size_t)nn);
    double *E = (double *)malloc(sizeof(double) * (size_t)nn * 3);
    double *Ep = (double *)malloc(sizeof(double) * (size_t)(np > 0 ? np : 1) * 3);
    oracle_deposit(n, L, np, xv, q, rho);
    oracle_solve_fft(n, L, rho, E);
    oracle_gather(n, L, np, xv, E, Ep);
    const double hk = -0.5 * (qm * dt);    /* v_{-1/2} = v_0 - (q/m) E dt/2 */
#pragma omp parallel for schedule(static) num_threads(g_threads)
    for (int64_t j = 0; j < np; ++j)
        for (int d = 0; d < 3; ++d)
            xv[(3 + d) * np + j] = fma(hk, Ep[d * np + j], xv[(3 + d) * np + j]);
    free(Ep);
    free(E);
    free(rho);
}

void oracle_run(int32_t n, double L, double dt, int64_t np, double *xv, int32_t nsteps,
                double *ex_energy, double *tot_energy, uint32_t *perm_last) {
    const int64_t nn = (int64_t)n * n * n;
    const double q = -((L * L) * L) / (double)np;
    const double qm_dt = -1.0 * dt;                  /* (q/m) dt, q/m = -1 */
    double *rho = (double *)malloc(sizeof(double) * (size_t)nn);
    double *E = (double *)malloc(sizeof(double) * (size_t)nn * 3);
    double *Ep = (double *)malloc(sizeof(double) * (size_t)(np > 0 ? np : 1) * 3);
    uint32_t *perm = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)(np > 0 ? np : 1));
    oracle_sort(n, L, np, xv, perm);                    /* canonical order */
    for (int32_t s = 0; s < nsteps; ++s) {
        oracle_deposit(n, L, np, xv, q, rho);           /* SCATTER */
        oracle_solve_fft(n, L, rho, E);                 /* SOLVE */
        double wx, w;
        oracle_field_energy(n, L, E, &wx, &w);
        if (ex_energy) ex_energy[s] = wx;
        if (tot_energy) tot_energy[s] = w;
        oracle_gather(n, L, np, xv, E, Ep);             /* GATHER */
        oracle_push(L, np, xv, Ep, qm_dt, dt);          /* PUSH + wrap */
        oracle_sort(n, L, np, xv, perm);                /* per-step sort by cell key */
    }
    if (perm_last && nsteps > 0) memcpy(perm_last, perm, sizeof(uint32_t) * (size_t)np);
    free(perm);
    free(Ep);
    free(E);
    free(rho);
}

/* ================================================= FD-PCG Poisson solve ==== *
 * P:179-181 (PCG solver: second-order central finite differences, matrix-free
 * CG), P:260 (SSOR preconditioner, four inner and two outer iterations,
 * damping factor pi/2; warm start from the previous time step)
 * (tolerance 1e-4).  Readings D#26-D#31: A = -Delta_h (7-point,
 * periodic), b = rho - mean(rho), red-black SSOR as `outer` x (`inner` forward
 * red/black sweeps, `inner` backward black/red sweeps) from z = 0, stopping
 * rule ||r||^2 <= tol^2 ||b||^2, E = -grad_h phi by central differences.
 * Node colour: red = (ix + iy + iz) even. */

/* y = A x = -Delta_h x: (6 x_m - sum of the six neighbours) / h^2. */
static double nb_sum(int32_t n, const double *x, int32_t ix, int32_t iy, int32_t iz) {
    return ((x[node(n, ix - 1, iy, iz)] + x[node(n, ix + 1, iy, iz)]) +
            (x[node(n, ix, iy - 1, iz)] + x[node(n, ix, iy + 1, iz)])) +
           (x[node(n, ix, iy, iz - 1)] + x[node(n, ix, iy, iz + 1)]);
}

void oracle_laplacian_fd(int32_t n, double L, const double *x, double *y) {
    const double inv_h = (double)n / L;
    const double ih2 = inv_h * inv_h;
    for (int32_t iz = 0; iz < n; ++iz)
        for (int32_t iy = 0; iy < n; ++iy)
            for (int32_t ix = 0; ix < n; ++ix) {
                int64_t m = node(n, ix, iy, iz);
                y[m] = (6.0 * x[m] - nb_sum(n, x, ix, iy, iz)) * ih2;
            }
}

/* One SOR half-sweep over the nodes of colour `colour` ("Gauss-Seidel",
 * P:260 damping factor omega): z_m <- (1 - omega) z_m + (omega/6)(h^2 r_m + sum nb z).
 * Every neighbour of a node has the other colour, so the order inside the colour
 * does not matter. */
static void sor_half_sweep(int32_t n, double h2, double c1, double c2, const double *r, double *z,
                           int colour) {
    for (int32_t iz = 0; iz < n; ++iz)
        for (int32_t iy = 0; iy < n; ++iy)
            for (int32_t ix = 0; ix < n; ++ix) {
                if (((ix + iy + iz) & 1) != colour) continue;
                int64_t m = node(n, ix, iy, iz);
                z[m] = c1 * z[m] + c2 * (h2 * r[m] + nb_sum(n, z, ix, iy, iz));
            }
}

/* z = M^-1 r, the SSOR preconditioner of P:260 (reading D#28): z = 0; outer times
 * { inner times (red, black) ; inner times (black, red) }.  The half-sweep sequence
 * is a palindrome, so M^-1 is symmetric (positive definite for 0 < omega < 2). */
void oracle_ssor(int32_t n, double L, const double *r, double *z, double omega, int32_t inner,
                 int32_t outer) {
    const int64_t nn = (int64_t)n * n * n;
    const double h = L / (double)n;
    const double h2 = h * h;
    const double c1 = 1.0 - omega, c2 = omega / 6.0;
    for (int64_t m = 0; m < nn; ++m) z[m] = 0.0;
    for (int32_t o = 0; o < outer; ++o) {
        for (int32_t i = 0; i < inner; ++i) {
            sor_half_sweep(n, h2, c1, c2, r, z, 0);
            sor_half_sweep(n, h2, c1, c2, r, z, 1);
        }
        for (int32_t i = 0; i < inner; ++i) {
            sor_half_sweep(n, h2, c1, c2, r, z, 1);
            sor_half_sweep(n, h2, c1, c2, r, z, 0);
        }
    }
}

static double dot(int64_t nn, const double *a, const double *b) {
    double s = 0.0;
    for (int64_t m = 0; m < nn; ++m) s += a[m] * b[m];
    return s;
}

/* Preconditioned CG (Saad Alg. 9.1) for A x = b from the initial guess in
 * x (warm start).  precond = 1: SSOR(omega, inner, outer); 0: none (M = I).
 * Stops when ||r||^2 <= tol^2 ||b||^2 (D#29); b = 0 gives x = 0.
 * Returns the iteration count, or -1 if maxit iterations did not converge. */
int32_t oracle_pcg(int32_t n, double L, const double *b, double *x, double tol, int32_t precond,
                   double omega, int32_t inner, int32_t outer, int32_t maxit, double *relres) {
    const int64_t nn = (int64_t)n * n * n;
    double *r = (double *)malloc(sizeof(double) * (size_t)nn);
    double *z = (double *)malloc(sizeof(double) * (size_t)nn);
    double *p = (double *)malloc(sizeof(double) * (size_t)nn);
    double *q = (double *)malloc(sizeof(double) * (size_t)nn);
    const double bb = dot(nn, b, b);
    const double stop = (tol * tol) * bb;
    int32_t it = 0, status = -1;
    double rr = 0.0;
    if (bb == 0.0) {
        for (int64_t m = 0; m < nn; ++m) x[m] = 0.0;
        status = 0;
        goto done;
    }
    oracle_laplacian_fd(n, L, x, q);                       /* r = b - A x */
    for (int64_t m = 0; m < nn; ++m) r[m] = b[m] - q[m];
    rr = dot(nn, r, r);
    if (rr <= stop) { status = 0; goto done; }
    if (precond) oracle_ssor(n, L, r, z, omega, inner, outer);
    else memcpy(z, r, sizeof(double) * (size_t)nn);
    memcpy(p, z, sizeof(double) * (size_t)nn);
    double rz = dot(nn, r, z);
    for (it = 1; it <= maxit; ++it) {
        oracle_laplacian_fd(n, L, p, q);                   /* q = A p */
        const double alpha = rz / dot(nn, p, q);
        for (int64_t m = 0; m < nn; ++m) x[m] = x[m] + alpha * p[m];
        for (int64_t m = 0; m < nn; ++m) r[m] = r[m] - alpha * q[m];
        rr = dot(nn, r, r);
        if (rr <= stop) { status = it; break; }
        if (precond) oracle_ssor(n, L, r, z, omega, inner, outer);
        else memcpy(z, r, sizeof(double) * (size_t)nn);
        const double rz_new = dot(nn, r, z);
        const double beta = rz_new / rz;
        rz = rz_new;
        for (int64_t m = 0; m < nn; ++m) p[m] = z[m] + beta * p[m];
    }
done:
    if (relres) *relres = bb > 0.0 ? sqrt(rr / bb) : 0.0;
    free(q);
    free(p);
    free(z);
    free(r);
    return status;
}

/* E = -grad_h phi by second-order central differences (D#30):
 * E_d(m) = (phi(m - e_d) - phi(m + e_d)) * (inv_h / 2). */
void oracle_gradient_central(int32_t n, double L, const double *phi, double *E) {
    const int64_t nn = (int64_t)n * n * n;
    const double c = 0.5 * ((double)n / L);
    for (int32_t iz = 0; iz < n; ++iz)
        for (int32_t iy = 0; iy < n; ++iy)
            for (int32_t ix = 0; ix < n; ++ix) {
                int64_t m = node(n, ix, iy, iz);
                E[m] = (phi[node(n, ix - 1, iy, iz)] - phi[node(n, ix + 1, iy, iz)]) * c;
                E[nn + m] = (phi[node(n, ix, iy - 1, iz)] - phi[node(n, ix, iy + 1, iz)]) * c;
                E[2 * nn + m] = (phi[node(n, ix, iy, iz - 1)] - phi[node(n, ix, iy, iz + 1)]) * c;
            }
}

/* The PCG solve of the PIC loop: b = rho - mean(rho) (ion background,
 * P:103, D#3), A phi = b by SSOR-PCG warm-started from phi, E = -grad_h phi.
 * Returns the iteration count (-1: not converged). */
int32_t oracle_solve_pcg(int32_t n, double L, const double *rho, double *phi, double *E, double tol,
                         double omega, int32_t inner, int32_t outer, int32_t maxit, double *relres) {
    const int64_t nn = (int64_t)n * n * n;
    double *b = (double *)malloc(sizeof(double) * (size_t)nn);
    double mean = 0.0;
    for (int64_t m = 0; m < nn; ++m) mean += rho[m];
    mean = mean / (double)nn;
    for (int64_t m = 0; m < nn; ++m) b[m] = rho[m] - mean;
    int32_t it = oracle_pcg(n, L, b, phi, tol, 1, omega, inner, outer, maxit, relres);
    oracle_gradient_central(n, L, phi, E);
    free(b);
    return it;
}

/* The PIC loop of oracle_run with the PCG solve in place of the FFT solve (BJ
 * config 5).  phi (N^3, in/out) is the warm start of the first solve and holds the
 * last solution on return; iters (nullable, nsteps) receives each solve's count. */
void oracle_run_pcg(int32_t n, double L, double dt, int64_t np, double *xv, int32_t nsteps,
                    double *ex_energy, double *tot_energy, double *phi, double tol, double omega,
                    int32_t inner, int32_t outer, int32_t maxit, int32_t *iters) {
    const int64_t nn = (int64_t)n * n * n;
    const double q = -((L * L) * L) / (double)np;
    const double qm_dt = -1.0 * dt;
    double *rho = (double *)malloc(sizeof(double) * (size_t)nn);
    double *E = (double *)malloc(sizeof(double) * (size_t)nn * 3);
    double *Ep = (double *)malloc(sizeof(double) * (size_t)(np > 0 ? np : 1) * 3);
    uint32_t *perm = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)(np > 0 ? np : 1));
    oracle_sort(n, L, np, xv, perm);
    for (int32_t s = 0; s < nsteps; ++s) {
        oracle_deposit(n, L, np, xv, q, rho);
        int32_t it = oracle_solve_pcg(n, L, rho, phi, E, tol, omega, inner, outer, maxit, NULL);
        if (iters) iters[s] = it;
        double wx, w;
        oracle_field_energy(n, L, E, &wx, &w);
        if (ex_energy) ex_energy[s] = wx;
        if (tot_energy) tot_energy[s] = w;
        oracle_gather(n, L, np, xv, E, Ep);
        oracle_push(L, np, xv, Ep, qm_dt, dt);
        oracle_sort(n, L, np, xv, perm);
    }
    free(perm);
    free(Ep);
    free(E);
    free(rho);
}

/* Backward half kick with the PCG field; phi (in/out) as in oracle_run_pcg. */
void oracle_half_kick_pcg(int32_t n, double L, double dt, int64_t np, double *xv, double *phi, double tol,
                          double omega, int32_t inner, int32_t outer, int32_t maxit) {
    const int64_t nn = (int64_t)n * n * n;
    const double q = -((L * L) * L) / (double)np;
    double *rho = (double *)malloc(sizeof(double) * (size_t)nn);
    double *E = (double *)malloc(sizeof(double) * (size_t)nn * 3);
    double *Ep = (double *)malloc(sizeof(double) * (size_t)(np > 0 ? np : 1) * 3);
    oracle_deposit(n, L, np, xv, q, rho);
    oracle_solve_pcg(n, L, rho, phi, E, tol, omega, inner, outer, maxit, NULL);
    oracle_gather(n, L, np, xv, E, Ep);
    const double hk = -0.5 * (-1.0 * dt);
    for (int64_t j = 0; j < np; ++j)
        for (int d = 0; d < 3; ++d)
            xv[(3 + d) * np + j] = fma(hk, Ep[d * np + j], xv[(3 + d) * np + j]);
    free(Ep);
    free(E);
    free(rho);
}

/* ================================== external fields and the Boris push ==== *
 * Eq. 1 / Eq. 3-4: dv/dt = (q/m)(E_int + E_ext + v x B_ext).
 * B_ext = 0: the leapfrog kick of oracle_push (bit for bit).  B_ext != 0: the Boris
 * scheme (half kick, rotation, half kick), reading D#32:
 *   hq = (q/m) dt / 2, t = hq B, s = 2 t / (1 + |t|^2),
 *   v- = v + hq E, v' = v- + v- x t, v+ = v- + v' x s, v <- v+ + hq E,
 * with E = E_p + E_ext (E_ext added only when nonzero), fma where written. */
static void cross3(const double a[3], const double b[3], double c[3]) {
    c[0] = a[1] * b[2] - a[2] * b[1];
    c[1] = a[2] * b[0] - a[0] * b[2];
    c[2] = a[0] * b[1] - a[1] * b[0];
}

void oracle_boris_coeffs(double dt, const double *b_ext, double t[3], double s[3]) {
    const double hq = 0.5 * (-1.0 * dt);   /* (q/m) dt / 2, q/m = -1 */
    for (int d = 0; d < 3; ++d) t[d] = hq * b_ext[d];
    const double tt = (t[0] * t[0] + t[1] * t[1]) + t[2] * t[2];
    for (int d = 0; d < 3; ++d) s[d] = (2.0 * t[d]) / (1.0 + tt);
}

void oracle_push_ext(double L, int64_t np, double *xv, const double *Ep, double dt, const double *b_ext,
                     const double *e_ext) {
    const double qm_dt = -1.0 * dt, hq = 0.5 * (-1.0 * dt);
    const int boris = b_ext && (b_ext[0] != 0.0 || b_ext[1] != 0.0 || b_ext[2] != 0.0);
    const int eext = e_ext && (e_ext[0] != 0.0 || e_ext[1] != 0.0 || e_ext[2] != 0.0);
    double t[3] = {0.0, 0.0, 0.0}, s[3] = {0.0, 0.0, 0.0};
    if (boris) oracle_boris_coeffs(dt, b_ext, t, s);
    for (int64_t j = 0; j < np; ++j) {
        double e[3], v[3];
        for (int d = 0; d < 3; ++d) {
            e[d] = eext ? Ep[d * np + j] + e_ext[d] : Ep[d * np + j];
            v[d] = xv[(3 + d) * np + j];
        }
        if (!boris) {
            for (int d = 0; d < 3; ++d) v[d] = fma(qm_dt, e[d], v[d]);
        } else {
            double vm[3], vp[3], vs[3], c[3];
            for (int d = 0; d < 3; ++d) vm[d] = fma(hq, e[d], v[d]);
            cross3(vm, t, c);
            for (int d = 0; d < 3; ++d) vp[d] = vm[d] + c[d];
            cross3(vp, s, c);
            for (int d = 0; d < 3; ++d) vs[d] = vm[d] + c[d];
            for (int d = 0; d < 3; ++d) v[d] = fma(hq, e[d], vs[d]);
        }
        for (int d = 0; d < 3; ++d) {
            xv[(3 + d) * np + j] = v[d];
            xv[d * np + j] = oracle_wrap(fma(v[d], dt, xv[d * np + j]), L);
        }
    }
}

void oracle_run_ext(int32_t n, double L, double dt, int64_t np, double *xv, int32_t nsteps,
                    double *ex_energy, double *tot_energy, const double *b_ext, const double *e_ext) {
    const int64_t nn = (int64_t)n * n * n;
    const double q = -((L * L) * L) / (double)np;
    double *rho = (double *)malloc(sizeof(double) * (size_t)nn);
    double *E = (double *)malloc(sizeof(double) * (size_t)nn * 3);
    double *Ep = (double *)malloc(sizeof(double) * (size_t)(np > 0 ? np : 1) * 3);
    uint32_t *perm = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)(np > 0 ? np : 1));
    oracle_sort(n, L, np, xv, perm);
    for (int32_t s = 0; s < nsteps; ++s) {
        oracle_deposit(n, L, np, xv, q, rho);
        oracle_solve_fft(n, L, rho, E);
        double wx, w;
        oracle_field_energy(n, L, E, &wx, &w);
        if (ex_energy) ex_energy[s] = wx;
        if (tot_energy) tot_energy[s] = w;
        oracle_gather(n, L, np, xv, E, Ep);
        oracle_push_ext(L, np, xv, Ep, dt, b_ext, e_ext);
        oracle_sort(n, L, np, xv, perm);
    }
    free(perm);
    free(Ep);
    free(E);
    free(rho);
}

/* ======================================== matrix-free Q1 FEM Poisson solve ==== *
 * P:183-195 (FEM with first-order Lagrange elements, matrix-free operator, CG;
 * plain CG for the comparison), P:226 (tol 1e-4), P:260 (warm start).
 * Readings D#33: element stiffness A^e_ij = int grad b_i . grad b_j over one cube
 * element by 2x2x2 Gauss quadrature; A x = sum_e scatter(A^e gather_e(x)) with the
 * periodic DOF map; lumped load b_j = h^3 rho_j minus its mean; E = -grad_h phi by
 * central differences (shared with the PCG path). */

/* A^e (8 x 8, vertex v = a + 2b + 4c at (a, b, c) h) by 2x2x2 Gauss-Legendre quadrature. */
void oracle_fem_element_stiffness(double h, double Ae[64]) {
    const double gp[2] = {0.5 - 0.5 / sqrt(3.0), 0.5 + 0.5 / sqrt(3.0)};   /* points on [0,1] */
    for (int i = 0; i < 64; ++i) Ae[i] = 0.0;
    for (int qz = 0; qz < 2; ++qz)
        for (int qy = 0; qy < 2; ++qy)
            for (int qx = 0; qx < 2; ++qx) {
                const double xi[3] = {gp[qx], gp[qy], gp[qz]};
                double grad[8][3];
                for (int v = 0; v < 8; ++v) {
                    const int a[3] = {v & 1, (v >> 1) & 1, (v >> 2) & 1};
                    double phi[3], dphi[3];
                    for (int d = 0; d < 3; ++d) {
                        phi[d] = a[d] ? xi[d] : 1.0 - xi[d];
                        dphi[d] = (a[d] ? 1.0 : -1.0) / h;           /* d/dx of the 1D basis */
                    }
                    grad[v][0] = dphi[0] * phi[1] * phi[2];
                    grad[v][1] = phi[0] * dphi[1] * phi[2];
                    grad[v][2] = phi[0] * phi[1] * dphi[2];
                }
                const double w = 0.125 * ((h * h) * h);              /* weight x Jacobian */
                for (int i = 0; i < 8; ++i)
                    for (int j = 0; j < 8; ++j)
                        Ae[i * 8 + j] += w * (grad[i][0] * grad[j][0] + grad[i][1] * grad[j][1] +
                                              grad[i][2] * grad[j][2]);
            }
}

/* y = A x, element by element ("the action of the matrix A"). */
void oracle_fem_apply(int32_t n, double L, const double *x, double *y) {
    const int64_t nn = (int64_t)n * n * n;
    double Ae[64];
    oracle_fem_element_stiffness(L / (double)n, Ae);
    for (int64_t m = 0; m < nn; ++m) y[m] = 0.0;
    for (int32_t ez = 0; ez < n; ++ez)
        for (int32_t ey = 0; ey < n; ++ey)
            for (int32_t ex = 0; ex < n; ++ex) {
                int64_t dof[8];
                double xe[8];
                for (int v = 0; v < 8; ++v) {
                    dof[v] = node(n, ex + (v & 1), ey + ((v >> 1) & 1), ez + ((v >> 2) & 1));
                    xe[v] = x[dof[v]];
                }
                for (int i = 0; i < 8; ++i) {
                    double s = 0.0;
                    for (int j = 0; j < 8; ++j) s += Ae[i * 8 + j] * xe[j];
                    y[dof[i]] += s;
                }
            }
}

/* Plain CG on A x = b from the guess in x; ||r||^2 <= tol^2 ||b||^2 (D#29). */
int32_t oracle_fem_cg(int32_t n, double L, const double *b, double *x, double tol, int32_t maxit,
                      double *relres) {
    const int64_t nn = (int64_t)n * n * n;
    double *r = (double *)malloc(sizeof(double) * (size_t)nn);
    double *p = (double *)malloc(sizeof(double) * (size_t)nn);
    double *q = (double *)malloc(sizeof(double) * (size_t)nn);
    const double bb = dot(nn, b, b), stop = (tol * tol) * bb;
    int32_t it = 0, status = -1;
    double rr = 0.0;
    if (bb == 0.0) {
        for (int64_t m = 0; m < nn; ++m) x[m] = 0.0;
        status = 0;
        goto done;
    }
    oracle_fem_apply(n, L, x, q);
    for (int64_t m = 0; m < nn; ++m) r[m] = b[m] - q[m];
    rr = dot(nn, r, r);
    if (rr <= stop) { status = 0; goto done; }
    memcpy(p, r, sizeof(double) * (size_t)nn);
    for (it = 1; it <= maxit; ++it) {
        oracle_fem_apply(n, L, p, q);
        const double alpha = rr / dot(nn, p, q);
        for (int64_t m = 0; m < nn; ++m) x[m] = x[m] + alpha * p[m];
        for (int64_t m = 0; m < nn; ++m) r[m] = r[m] - alpha * q[m];
        const double rr_new = dot(nn, r, r);
        if (rr_new <= stop) { rr = rr_new; status = it; break; }
        const double beta = rr_new / rr;
        rr = rr_new;
        for (int64_t m = 0; m < nn; ++m) p[m] = r[m] + beta * p[m];
    }
done:
    if (relres) *relres = bb > 0.0 ? sqrt(rr / bb) : 0.0;
    free(q);
    free(p);
    free(r);
    return status;
}

/* The FEM solve of the PIC loop: b_j = h^3 rho_j - mean, CG warm-started from phi,
 * E = -grad_h phi (central differences).  Returns the iteration count (-1: not converged). */
int32_t oracle_solve_fem(int32_t n, double L, const double *rho, double *phi, double *E, double tol,
                         int32_t maxit, double *relres) {
    const int64_t nn = (int64_t)n * n * n;
    const double h = L / (double)n, h3 = (h * h) * h;
    double *b = (double *)malloc(sizeof(double) * (size_t)nn);
    double mean = 0.0;
    for (int64_t m = 0; m < nn; ++m) {
        b[m] = h3 * rho[m];
        mean += b[m];
    }
    mean = mean / (double)nn;
    for (int64_t m = 0; m < nn; ++m) b[m] = b[m] - mean;
    int32_t it = oracle_fem_cg(n, L, b, phi, tol, maxit, relres);
    oracle_gradient_central(n, L, phi, E);
    free(b);
    return it;
}

/* oracle_run with the FEM solve; phi in/out (warm start); iters (nullable) per step. */
void oracle_run_fem(int32_t n, double L, double dt, int64_t np, double *xv, int32_t nsteps,
                    double *ex_energy, double *tot_energy, double *phi, double tol, int32_t maxit,
                    int32_t *iters) {
    const int64_t nn = (int64_t)n * n * n;
    const double q = -((L * L) * L) / (double)np;
    const double qm_dt = -1.0 * dt;
    double *rho = (double *)malloc(sizeof(double) * (size_t)nn);
    double *E = (double *)malloc(sizeof(double) * (size_t)nn * 3);
    double *Ep = (double *)malloc(sizeof(double) * (size_t)(np > 0 ? np : 1) * 3);
    uint32_t *perm = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)(np > 0 ? np : 1));
    oracle_sort(n, L, np, xv, perm);
    for (int32_t s = 0; s < nsteps; ++s) {
        oracle_deposit(n, L, np, xv, q, rho);
        int32_t it = oracle_solve_fem(n, L, rho, phi, E, tol, maxit, NULL);
        if (iters) iters[s] = it;
        double wx, w;
        oracle_field_energy(n, L, E, &wx, &w);
        if (ex_energy) ex_energy[s] = wx;
        if (tot_energy) tot_energy[s] = w;
        oracle_gather(n, L, np, xv, E, Ep);
        oracle_push(L, np, xv, Ep, qm_dt, dt);
        oracle_sort(n, L, np, xv, perm);
    }
    free(perm);
    free(Ep);
    free(E);
    free(rho);
}

/* Backward half kick with the FEM field; phi (in/out) as in oracle_run_fem. */
void oracle_half_kick_fem(int32_t n, double L, double dt, int64_t np, double *xv, double *phi, double tol,
                          int32_t maxit) {
    const int64_t nn = (int64_t)n * n * n;
    const double q = -((L * L) * L) / (double)np;
    double *rho = (double *)malloc(sizeof(double) * (size_t)nn);
    double *E = (double *)malloc(sizeof(double) * (size_t)nn * 3);
    double *Ep = (double *)malloc(sizeof(double) * (size_t)(np > 0 ? np : 1) * 3);
    oracle_deposit(n, L, np, xv, q, rho);
    oracle_solve_fem(n, L, rho, phi, E, tol, maxit, NULL);
    oracle_gather(n, L, np, xv, E, Ep);
    const double hk = -0.5 * (-1.0 * dt);
    for (int64_t j = 0; j < np; ++j)
        for (int d = 0; d < 3; ++d)
            xv[(3 + d) * np + j] = fma(hk, Ep[d * np + j], xv[(3 + d) * np + j]);
    free(Ep);
    free(E);
    free(rho);
}
