// pic_api.cu -- C ABI (include/pic.h) and the host-side orchestration of the
// PIC step.  The host validates, carves the caller's workspace and enqueues
// kernels on the caller's stream; every step of the path runs on the device
// (kernels.h).  One step:
//   SOLVE   fft_x_fwd -> fft_y_fwd -> fft_z_mul -> fft_y_inv -> fft_x_inv (E4) -> energy
//   CLEAR   count = 0, rho = 0
//   PUSH    push_key  (gather + push + new key + count)
//   SORT    scan -> place
//   SCATTER reorder_deposit (sorted gather + push + stream out + CIC deposit)
#include <cmath>
#include <cstdio>
#include <cstring>
#include <new>
#include <vector>

#include "../../include/pic.h"
#include "kernels.h"

namespace pic {
void fft_set_smem_limits();
void particles_set_smem_limits();
}

using pic::Geom;
using pic::PState;

namespace {

thread_local char g_init_error[512] = "";
constexpr int kMaxEnergySteps = 4096;   // device ring of per-step (W_x, W)

const char* kStageNames[PIC_NSTAGES] = {
    "fft_x_fwd", "fft_y_fwd", "fft_z_mul", "fft_y_inv", "fft_x_inv", "energy",
    "clear",     "push_key",  "scan",      "place",     "reorder_deposit"};

size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

bool is_pow2(int v) { return v > 0 && (v & (v - 1)) == 0; }

}  // namespace

struct pic_ctx {
    pic_params p{};
    Geom g{};
    int64_t np = 0;
    int64_t ncell = 0;
    double q = 0.0;               // macro charge -L^3 / N_p
    double deposit_scale = 0.0;   // q inv_h^3 (raw CIC weight sums -> rho)
    cudaStream_t stream = nullptr;
    bool poisoned = false;
    char err[512] = "";
    double2* part[2][3] = {};     // double-buffered pair streams (pic_device.cuh)
    int cur = 0;
    uint32_t* key = nullptr;
    uint16_t* rank = nullptr;     // arrival order of each particle in its new cell
    uint32_t* perm = nullptr;
    uint32_t* count = nullptr;
    uint32_t* offs = nullptr;
    uint32_t* scan_scratch = nullptr;
    double* rho = nullptr;        // S0: pitched raw CIC weight sums / spectrum during the solve
    double* spec[2] = {};         // S1, S2: half spectra of E_x, E_y during the solve
    double* E4 = nullptr;         // field node records (E_x, E_y, E_z, 0)
    double2* tw = nullptr;
    double* partials = nullptr;
    double* energies = nullptr;   // ring [kMaxEnergySteps][2]
    int* err_flag = nullptr;
    int last_slot = -1;
    // timing
    bool timing = false;
    double stage_ms[PIC_NSTAGES] = {};
    int64_t stage_launches[PIC_NSTAGES] = {};
    std::vector<cudaEvent_t> ev_pool;
    std::vector<int> ev_stage;    // stage of pending pair k (events 2k, 2k+1)
    size_t ev_used = 0;           // pairs in use
};

namespace {

// ------------------------------------------------------------ validation ---
pic_status validate(const pic_params* p, int32_t rank, int32_t nranks, char* msg, size_t msz) {
    if (!p) { snprintf(msg, msz, "params is NULL"); return PIC_EINVAL; }
    if (nranks != 1 || rank != 0) {
        snprintf(msg, msz, "nranks=%d rank=%d: this build runs one rank (nranks == 1)", nranks, rank);
        return nranks < 1 || rank < 0 || rank >= nranks ? PIC_EINVAL : PIC_EUNSUPPORTED;
    }
    if (p->pgrid[0] != 1 || p->pgrid[1] != 1) { snprintf(msg, msz, "pgrid must be {1,1}"); return PIC_EINVAL; }
    if (!is_pow2(p->n) || p->n < 16 || p->n > 1024) { snprintf(msg, msz, "n=%d: power of two in [16,1024]", p->n); return PIC_EINVAL; }
    if (p->ppc <= 0 || p->ppc > 1024) { snprintf(msg, msz, "ppc=%d: must be in [1,1024]", p->ppc); return PIC_EINVAL; }
    if (!(p->k > 0) || !std::isfinite(p->k)) { snprintf(msg, msz, "k must be > 0"); return PIC_EINVAL; }
    if (!(p->alpha >= 0 && p->alpha < 1)) { snprintf(msg, msz, "alpha=%g: need 0 <= alpha < 1", p->alpha); return PIC_EINVAL; }
    if (!(p->dt > 0) || !std::isfinite(p->dt)) { snprintf(msg, msz, "dt must be > 0"); return PIC_EINVAL; }
    const double L = p->length == 0.0 ? 2.0 * M_PI / p->k : p->length;
    if (!(L > 0) || !std::isfinite(L)) { snprintf(msg, msz, "length must be > 0"); return PIC_EINVAL; }
    const double m = p->k * L / (2.0 * M_PI);
    if (std::fabs(m - std::round(m)) > 1e-9 * std::max(1.0, m) || std::round(m) < 1) {
        snprintf(msg, msz, "k L / 2 pi = %g must be a positive integer", m);
        return PIC_EINVAL;
    }
    const double np = (double)p->ppc * p->n * p->n * p->n;
    if (np >= 4294967296.0) { snprintf(msg, msz, "N_p = %.0f >= 2^32 on one rank", np); return PIC_EINVAL; }
    return PIC_OK;
}

Geom make_geom(const pic_params* p) {
    Geom g{};
    g.n = p->n;
    g.nmask = p->n - 1;
    g.px = (int)align_up((size_t)(p->n / 2 + 1), 8);
    g.rp = 2 * g.px;
    g.L = p->length == 0.0 ? 2.0 * M_PI / p->k : p->length;
    g.inv_h = (double)p->n / g.L;
    g.dt = p->dt;
    g.qm_dt = -1.0 * p->dt;     // q/m = -1
    return g;
}

// Carve the workspace; returns the bytes needed (pointers set when c != nullptr).
size_t carve(pic_ctx* c, const Geom& g, int64_t np, char* base) {
    size_t off = 0;
    auto take = [&](size_t bytes) -> char* {
        off = align_up(off, 256);
        char* ptr = base ? base + off : nullptr;
        off += bytes;
        return ptr;
    };
    const int64_t ncell = (int64_t)g.n * g.n * g.n;
    const size_t grid_bytes = sizeof(double2) * (size_t)g.n * g.n * g.px;
    for (int b = 0; b < 2; ++b)
        for (int a = 0; a < 3; ++a) {
            char* ptr = take(sizeof(double2) * (size_t)np);
            if (c) c->part[b][a] = reinterpret_cast<double2*>(ptr);
        }
    char* k = take(sizeof(uint32_t) * (size_t)np);
    char* rk = take(sizeof(uint16_t) * (size_t)np);
    char* pm = take(sizeof(uint32_t) * (size_t)np);
    char* cn = take(sizeof(uint32_t) * (size_t)ncell);
    char* of = take(sizeof(uint32_t) * (size_t)(ncell + 1));
    char* ss = take(pic::scan_scratch_bytes(ncell));
    char* rh = take(grid_bytes);
    char* s1 = take(grid_bytes);
    char* s2 = take(grid_bytes);
    char* e4 = take(sizeof(double) * 4 * (size_t)ncell);
    char* tw = take(sizeof(double2) * (size_t)g.n);
    char* pa = take(sizeof(double) * 3 * (size_t)pic::energy_partials(g));
    char* en = take(sizeof(double) * 2 * kMaxEnergySteps);
    char* ef = take(sizeof(int) * 4);
    if (c) {
        c->key = reinterpret_cast<uint32_t*>(k);
        c->rank = reinterpret_cast<uint16_t*>(rk);
        c->perm = reinterpret_cast<uint32_t*>(pm);
        c->count = reinterpret_cast<uint32_t*>(cn);
        c->offs = reinterpret_cast<uint32_t*>(of);
        c->scan_scratch = reinterpret_cast<uint32_t*>(ss);
        c->rho = reinterpret_cast<double*>(rh);
        c->spec[0] = reinterpret_cast<double*>(s1);
        c->spec[1] = reinterpret_cast<double*>(s2);
        c->E4 = reinterpret_cast<double*>(e4);
        c->tw = reinterpret_cast<double2*>(tw);
        c->partials = reinterpret_cast<double*>(pa);
        c->energies = reinterpret_cast<double*>(en);
        c->err_flag = reinterpret_cast<int*>(ef);
    }
    return align_up(off, 256);
}

pic_status fail(pic_ctx* c, pic_status st, const char* what, cudaError_t e = cudaSuccess) {
    if (e != cudaSuccess)
        snprintf(c->err, sizeof(c->err), "%s: %s", what, cudaGetErrorString(e));
    else
        snprintf(c->err, sizeof(c->err), "%s", what);
    if (st == PIC_ECUDA) c->poisoned = true;
    return st;
}

#define PIC_CUDA(ctx, call)                                              \
    do {                                                                 \
        cudaError_t e_ = (call);                                         \
        if (e_ != cudaSuccess) return fail((ctx), PIC_ECUDA, #call, e_); \
    } while (0)

#define PIC_LAUNCHED(ctx, what)                                          \
    do {                                                                 \
        cudaError_t e_ = cudaGetLastError();                             \
        if (e_ != cudaSuccess) return fail((ctx), PIC_ECUDA, what, e_);  \
    } while (0)

// ---------------------------------------------------------------- timing ---
struct StageScope {
    pic_ctx* c;
    int stage;
    size_t pair;
    StageScope(pic_ctx* ctx, int st, int nlaunch) : c(ctx), stage(st), pair(0) {
        if (!c->timing) return;
        pair = c->ev_used++;
        if (c->ev_pool.size() < 2 * c->ev_used) {
            for (int q = 0; q < 2; ++q) {
                cudaEvent_t e;
                cudaEventCreate(&e);
                c->ev_pool.push_back(e);
            }
            c->ev_stage.push_back(0);
        }
        c->ev_stage[pair] = st;
        c->stage_launches[st] += nlaunch;
        cudaEventRecord(c->ev_pool[2 * pair], c->stream);
    }
    ~StageScope() {
        if (c->timing) cudaEventRecord(c->ev_pool[2 * pair + 1], c->stream);
    }
};

void collect_timings(pic_ctx* c) {
    for (size_t k = 0; k < c->ev_used; ++k) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, c->ev_pool[2 * k], c->ev_pool[2 * k + 1]) == cudaSuccess)
            c->stage_ms[c->ev_stage[k]] += ms;
    }
    c->ev_used = 0;
}

// ------------------------------------------------------------ pipeline -----
PState state(pic_ctx* c, int b) {
    PState s;
    for (int a = 0; a < 3; ++a) s.p[a] = c->part[b][a];
    return s;
}

// rho (raw CIC sums, scaled by `scale` in the multiply) -> E, energies -> ring slot
pic_status solve(pic_ctx* c, double scale, int slot) {
    const Geom& g = c->g;
    double* const S[3] = {c->spec[0], c->spec[1], c->rho};   // E^_x, E^_y, E^_z after the z pass
    double* const S0[3] = {c->rho, c->rho, c->rho};
    { StageScope t(c, PIC_STAGE_FFT_X_FWD, 1); pic::launch_fft_x_fwd(g, c->rho, c->tw, c->stream); }
    PIC_LAUNCHED(c, "fft_x_fwd");
    { StageScope t(c, PIC_STAGE_FFT_Y_FWD, 1); pic::launch_fft_y(g, S0, 1, 0, c->tw, c->stream); }
    PIC_LAUNCHED(c, "fft_y_fwd");
    { StageScope t(c, PIC_STAGE_FFT_Z_MUL, 1); pic::launch_fft_z_mul(g, c->rho, c->spec[0], c->spec[1], scale, c->tw, c->stream); }
    PIC_LAUNCHED(c, "fft_z_mul");
    { StageScope t(c, PIC_STAGE_FFT_Y_INV, 1); pic::launch_fft_y(g, S, 3, 1, c->tw, c->stream); }
    PIC_LAUNCHED(c, "fft_y_inv");
    { StageScope t(c, PIC_STAGE_FFT_X_INV, 1); pic::launch_fft_x_inv(g, S, c->E4, c->tw, c->partials, c->stream); }
    PIC_LAUNCHED(c, "fft_x_inv");
    { StageScope t(c, PIC_STAGE_ENERGY, 1); pic::launch_energy_reduce(g, c->partials, c->energies + 2 * slot, c->stream); }
    PIC_LAUNCHED(c, "energy");
    c->last_slot = slot;
    return PIC_OK;
}

// (optionally pushed) particles of buffer cur -> sorted by key into cur^1, rho
// deposited; cur flips.
pic_status push_sort_deposit(pic_ctx* c, int push) {
    const Geom& g = c->g;
    {
        StageScope t(c, PIC_STAGE_CLEAR, 0);
        PIC_CUDA(c, cudaMemsetAsync(c->count, 0, sizeof(uint32_t) * (size_t)c->ncell, c->stream));
        PIC_CUDA(c, cudaMemsetAsync(c->rho, 0, sizeof(double2) * (size_t)g.n * g.n * g.px, c->stream));
    }
    PState cur = state(c, c->cur), nxt = state(c, c->cur ^ 1);
    { StageScope t(c, PIC_STAGE_PUSH_KEY, 1); pic::launch_push_key(g, cur, c->np, c->offs, c->E4, push, c->key, c->rank, c->count, c->err_flag, c->stream); }
    PIC_LAUNCHED(c, "push_key");
    { StageScope t(c, PIC_STAGE_SCAN, 3); pic::launch_scan(c->count, c->offs, c->ncell, c->scan_scratch, c->stream); }
    PIC_LAUNCHED(c, "scan");
    { StageScope t(c, PIC_STAGE_PLACE, 1); pic::launch_place(c->key, c->rank, c->np, c->offs, c->perm, c->stream); }
    PIC_LAUNCHED(c, "place");
    {
        StageScope t(c, PIC_STAGE_REORDER_DEPOSIT, 1);
        pic::launch_reorder_deposit(g, c->offs, c->perm, cur, nxt, push, c->rho, c->err_flag, c->stream);
    }
    PIC_LAUNCHED(c, "reorder_deposit");
    c->cur ^= 1;
    return PIC_OK;
}

pic_status sync_check(pic_ctx* c) {
    PIC_CUDA(c, cudaStreamSynchronize(c->stream));
    int flag[2] = {0, 0};
    PIC_CUDA(c, cudaMemcpy(flag, c->err_flag, sizeof(flag), cudaMemcpyDeviceToHost));
    if (flag[1]) {
        PIC_CUDA(c, cudaMemset(c->err_flag + 1, 0, sizeof(int)));
        return fail(c, PIC_EINVAL, "imported position outside [0, L); particle state undefined");
    }
    if (flag[0]) return fail(c, PIC_EOVERFLOW, "a cell holds more particles than one chunk (4096) or 65535");
    if (c->timing) collect_timings(c);
    return PIC_OK;
}

pic_status copy_grid_to_device(pic_ctx* c, double* dst, const double* host) {
    const Geom& g = c->g;
    PIC_CUDA(c, cudaMemcpy2DAsync(dst, sizeof(double) * g.rp, host, sizeof(double) * g.n,
                                  sizeof(double) * g.n, (size_t)g.n * g.n, cudaMemcpyHostToDevice,
                                  c->stream));
    return PIC_OK;
}

pic_status copy_grid_to_host(pic_ctx* c, double* host, const double* src) {
    const Geom& g = c->g;
    PIC_CUDA(c, cudaMemcpy2DAsync(host, sizeof(double) * g.n, src, sizeof(double) * g.rp,
                                  sizeof(double) * g.n, (size_t)g.n * g.n, cudaMemcpyDeviceToHost,
                                  c->stream));
    return PIC_OK;
}

#define PIC_TRY(expr)                       \
    do {                                    \
        pic_status s_ = (expr);             \
        if (s_ != PIC_OK) return s_;        \
    } while (0)

#define PIC_CHECK_CTX(c)                                 \
    do {                                                 \
        if (!(c)) return PIC_EINVAL;                     \
        if ((c)->poisoned) return PIC_EPOISONED;         \
    } while (0)

}  // namespace

// ================================================================== ABI ====
extern "C" {

pic_status pic_params_default(pic_params* p) {
    if (!p) return PIC_EINVAL;
    std::memset(p, 0, sizeof(*p));
    p->n = 16;
    p->ppc = 8;
    p->k = 0.5;
    p->length = 0.0;
    p->alpha = 0.05;
    p->dt = 0.05;
    p->seed = 1;
    p->half_kick = 1;
    p->pgrid[0] = 1;
    p->pgrid[1] = 1;
    return PIC_OK;
}

pic_status pic_workspace_bytes(const pic_params* p, int32_t rank, int32_t nranks, size_t* bytes) {
    char msg[256];
    pic_status st = validate(p, rank, nranks, msg, sizeof(msg));
    if (st != PIC_OK) { snprintf(g_init_error, sizeof(g_init_error), "%s", msg); return st; }
    if (!bytes) return PIC_EINVAL;
    const Geom g = make_geom(p);
    const int64_t np = (int64_t)p->ppc * p->n * p->n * p->n;
    *bytes = carve(nullptr, g, np, nullptr);
    return PIC_OK;
}

pic_status pic_init(const pic_params* p, int32_t rank, int32_t nranks, const uint8_t* nccl_id,
                    void* workspace, size_t workspace_bytes, void* cuda_stream, pic_ctx** out) {
    (void)nccl_id;
    if (!out) return PIC_EINVAL;
    *out = nullptr;
    char msg[256];
    pic_status st = validate(p, rank, nranks, msg, sizeof(msg));
    if (st != PIC_OK) { snprintf(g_init_error, sizeof(g_init_error), "%s", msg); return st; }
    const Geom g = make_geom(p);
    const int64_t np = (int64_t)p->ppc * p->n * p->n * p->n;
    const size_t need = carve(nullptr, g, np, nullptr);
    if (!workspace || workspace_bytes < need) {
        snprintf(g_init_error, sizeof(g_init_error), "workspace %zu B < %zu B needed", workspace_bytes, need);
        return PIC_ENOMEM;
    }
    pic_ctx* c = new (std::nothrow) pic_ctx();
    if (!c) return PIC_ENOMEM;
    c->p = *p;
    c->g = g;
    c->np = np;
    c->ncell = (int64_t)g.n * g.n * g.n;
    c->q = -((g.L * g.L) * g.L) / (double)np;
    c->deposit_scale = c->q * ((g.inv_h * g.inv_h) * g.inv_h);
    c->stream = reinterpret_cast<cudaStream_t>(cuda_stream);
    carve(c, g, np, reinterpret_cast<char*>(workspace));

    static bool smem_set = false;
    if (!smem_set) { pic::fft_set_smem_limits(); pic::particles_set_smem_limits(); smem_set = true; }

    auto bail = [&](pic_status s) {
        snprintf(g_init_error, sizeof(g_init_error), "%s", c->err);
        delete c;
        return s;
    };
    // twiddles W_n^m = exp(-2 pi i m / n), m < n/2
    std::vector<double2> tw(g.n);   // W_n^m = exp(-2 pi i m / n), m < n
    for (int m = 0; m < g.n; ++m) {
        const double ang = 2.0 * M_PI * (double)m / (double)g.n;
        tw[m] = make_double2(std::cos(ang), -std::sin(ang));
    }
    cudaError_t e = cudaMemcpyAsync(c->tw, tw.data(), sizeof(double2) * tw.size(), cudaMemcpyHostToDevice, c->stream);
    if (e == cudaSuccess) e = cudaMemsetAsync(c->err_flag, 0, sizeof(int) * 4, c->stream);
    if (e != cudaSuccess) return bail(fail(c, PIC_ECUDA, "init copies", e));

    pic::launch_sample(g, state(c, 0), np, p->k, p->alpha, p->seed, c->stream);
    e = cudaGetLastError();
    if (e != cudaSuccess) return bail(fail(c, PIC_ECUDA, "sample", e));
    c->cur = 0;
    if ((st = push_sort_deposit(c, 0)) != PIC_OK) return bail(st);
    if (p->half_kick) {
        if ((st = solve(c, c->deposit_scale / (double)c->ncell, 0)) != PIC_OK) return bail(st);
        pic::launch_half_kick(g, state(c, c->cur), np, c->E4, c->stream);
        e = cudaGetLastError();
        if (e != cudaSuccess) return bail(fail(c, PIC_ECUDA, "half_kick", e));
        c->last_slot = -1;
        // the solve reused the charge buffer: deposit again (the re-sort is the identity)
        if ((st = push_sort_deposit(c, 0)) != PIC_OK) return bail(st);
    }
    if ((st = sync_check(c)) != PIC_OK) return bail(st);
    *out = c;
    return PIC_OK;
}

pic_status pic_step(pic_ctx* c, int32_t nsteps, double* ex_energy) {
    PIC_CHECK_CTX(c);
    if (nsteps < 0) return PIC_EINVAL;
    const double scale = c->deposit_scale / (double)c->ncell;
    int32_t done = 0;
    while (done < nsteps) {
        const int chunk = std::min(nsteps - done, kMaxEnergySteps);
        for (int s = 0; s < chunk; ++s) {
            PIC_TRY(solve(c, scale, s));
            PIC_TRY(push_sort_deposit(c, 1));
        }
        std::vector<double> en(2 * (size_t)chunk);
        PIC_CUDA(c, cudaMemcpyAsync(en.data(), c->energies, sizeof(double) * en.size(),
                                    cudaMemcpyDeviceToHost, c->stream));
        PIC_TRY(sync_check(c));
        for (int s = 0; s < chunk; ++s) {
            if (!std::isfinite(en[2 * s]) || !std::isfinite(en[2 * s + 1]))
                return fail(c, PIC_ENONFINITE, "non-finite field energy");
            if (ex_energy) ex_energy[done + s] = en[2 * s];
        }
        done += chunk;
    }
    return PIC_OK;
}

pic_status pic_field_energy(pic_ctx* c, double* ex_energy, double* total_energy) {
    PIC_CHECK_CTX(c);
    if (c->last_slot < 0) { snprintf(c->err, sizeof(c->err), "no solve yet"); return PIC_EINVAL; }
    double en[2];
    PIC_CUDA(c, cudaMemcpyAsync(en, c->energies + 2 * c->last_slot, sizeof(en), cudaMemcpyDeviceToHost, c->stream));
    PIC_TRY(sync_check(c));
    if (ex_energy) *ex_energy = en[0];
    if (total_energy) *total_energy = en[1];
    return PIC_OK;
}

void pic_free(pic_ctx* c) {
    if (!c) return;
    if (c->stream) cudaStreamSynchronize(c->stream);
    for (cudaEvent_t e : c->ev_pool) cudaEventDestroy(e);
    delete c;
}

const char* pic_last_error(const pic_ctx* c) { return c ? c->err : g_init_error; }

pic_status pic_num_particles(pic_ctx* c, int64_t* np) {
    if (!c || !np) return PIC_EINVAL;
    *np = c->np;
    return PIC_OK;
}

pic_status pic_get_particles(pic_ctx* c, double* xyzuvw, int64_t np) {
    PIC_CHECK_CTX(c);
    if (!xyzuvw || np != c->np) return PIC_EINVAL;
    // the idle buffer (48 B/particle) holds the SoA [6][np] copy for the transfer
    double* soa = reinterpret_cast<double*>(c->part[c->cur ^ 1][0]);
    pic::launch_pairs_to_soa(state(c, c->cur), np, soa, c->stream);
    PIC_LAUNCHED(c, "pairs_to_soa");
    PIC_CUDA(c, cudaMemcpyAsync(xyzuvw, soa, sizeof(double) * 6 * (size_t)np, cudaMemcpyDeviceToHost, c->stream));
    return sync_check(c);
}

pic_status pic_set_particles(pic_ctx* c, const double* xyzuvw, int64_t np) {
    PIC_CHECK_CTX(c);
    if (!xyzuvw || np != c->np) return PIC_EINVAL;
    double* soa = reinterpret_cast<double*>(c->part[c->cur ^ 1][0]);
    PIC_CUDA(c, cudaMemcpyAsync(soa, xyzuvw, sizeof(double) * 6 * (size_t)np, cudaMemcpyHostToDevice, c->stream));
    pic::launch_soa_to_pairs(soa, np, state(c, c->cur), c->stream);
    PIC_LAUNCHED(c, "soa_to_pairs");
    PIC_TRY(push_sort_deposit(c, 0));
    c->last_slot = -1;
    return sync_check(c);
}

pic_status pic_get_grid(pic_ctx* c, int32_t which, double* host) {
    PIC_CHECK_CTX(c);
    if (!host || which < 0 || which > 3) return PIC_EINVAL;
    if (which == 0) {
        PIC_TRY(copy_grid_to_host(c, host, c->rho));
    } else {
        pic::launch_e4_extract(c->g, c->E4, which - 1, c->spec[0], c->stream);   // S1 as scratch
        PIC_LAUNCHED(c, "e4_extract");
        PIC_CUDA(c, cudaMemcpyAsync(host, c->spec[0], sizeof(double) * (size_t)c->ncell,
                                    cudaMemcpyDeviceToHost, c->stream));
    }
    PIC_TRY(sync_check(c));
    if (which == 0)
        for (int64_t m = 0; m < c->ncell; ++m) host[m] = c->deposit_scale * host[m];
    return PIC_OK;
}

pic_status pic_solve_injected(pic_ctx* c, const double* rho_host, double* E_host, double* ex_energy,
                              double* total_energy) {
    PIC_CHECK_CTX(c);
    if (!rho_host) return PIC_EINVAL;
    PIC_TRY(copy_grid_to_device(c, c->rho, rho_host));
    PIC_TRY(solve(c, 1.0 / (double)c->ncell, 0));
    double en[2];
    PIC_CUDA(c, cudaMemcpyAsync(en, c->energies, sizeof(en), cudaMemcpyDeviceToHost, c->stream));
    if (E_host)
        for (int d = 0; d < 3; ++d) {
            pic::launch_e4_extract(c->g, c->E4, d, c->spec[0], c->stream);
            PIC_LAUNCHED(c, "e4_extract");
            PIC_CUDA(c, cudaMemcpyAsync(E_host + (size_t)d * c->ncell, c->spec[0], sizeof(double) * (size_t)c->ncell,
                                        cudaMemcpyDeviceToHost, c->stream));
        }
    PIC_TRY(sync_check(c));
    if (ex_energy) *ex_energy = en[0];
    if (total_energy) *total_energy = en[1];
    // restore the charge of the particles (re-sort is the identity: already sorted)
    PIC_TRY(push_sort_deposit(c, 0));
    c->last_slot = -1;
    return sync_check(c);
}

pic_status pic_push_injected(pic_ctx* c, const double* E_host) {
    PIC_CHECK_CTX(c);
    if (!E_host) return PIC_EINVAL;
    double* const comp[3] = {c->spec[0], c->spec[1], c->rho};   // scratch: compact [n^3] each
    for (int d = 0; d < 3; ++d)
        PIC_CUDA(c, cudaMemcpyAsync(comp[d], E_host + (size_t)d * c->ncell, sizeof(double) * (size_t)c->ncell,
                                    cudaMemcpyHostToDevice, c->stream));
    pic::launch_e4_pack(c->g, comp, c->E4, c->stream);
    PIC_LAUNCHED(c, "e4_pack");
    PIC_TRY(push_sort_deposit(c, 1));
    c->last_slot = -1;
    return sync_check(c);
}

pic_status pic_get_keys_perm(pic_ctx* c, uint32_t* keys, uint32_t* perm) {
    PIC_CHECK_CTX(c);
    if (perm) {
        pic::launch_sort_segments(c->offs, c->ncell, c->perm, c->stream);
        PIC_LAUNCHED(c, "sort_segments");
        PIC_CUDA(c, cudaMemcpyAsync(perm, c->perm, sizeof(uint32_t) * (size_t)c->np, cudaMemcpyDeviceToHost, c->stream));
    }
    PIC_TRY(sync_check(c));
    if (keys) {
        pic::launch_keys_only(c->g, state(c, c->cur), c->np, c->key, c->stream);
        PIC_LAUNCHED(c, "keys_only");
        PIC_CUDA(c, cudaMemcpyAsync(keys, c->key, sizeof(uint32_t) * (size_t)c->np, cudaMemcpyDeviceToHost, c->stream));
        PIC_TRY(sync_check(c));
    }
    return PIC_OK;
}

pic_status pic_set_timing(pic_ctx* c, int32_t enable) {
    PIC_CHECK_CTX(c);
    PIC_TRY(sync_check(c));
    c->timing = enable != 0;
    return PIC_OK;
}

pic_status pic_get_timings(pic_ctx* c, double* ms, int64_t* launches) {
    PIC_CHECK_CTX(c);
    PIC_TRY(sync_check(c));
    for (int s = 0; s < PIC_NSTAGES; ++s) {
        if (ms) ms[s] = c->stage_ms[s];
        if (launches) launches[s] = c->stage_launches[s];
    }
    return PIC_OK;
}

pic_status pic_reset_timings(pic_ctx* c) {
    PIC_CHECK_CTX(c);
    PIC_TRY(sync_check(c));
    for (int s = 0; s < PIC_NSTAGES; ++s) { c->stage_ms[s] = 0.0; c->stage_launches[s] = 0; }
    return PIC_OK;
}

const char* pic_stage_name(int32_t stage) {
    return stage >= 0 && stage < PIC_NSTAGES ? kStageNames[stage] : nullptr;
}

pic_status pic_launches_per_step(pic_ctx* c, int64_t* launches) {
    if (!c || !launches) return PIC_EINVAL;
    *launches = 6 /* solve */ + 1 /* push_key */ + 3 /* scan */ + 1 /* place */ + 1 /* reorder_deposit */;
    return PIC_OK;
}

}  // extern "C"
