// pic_api.cu -- C ABI (include/pic.h) and the host-side orchestration of the
// PIC step.  The host validates, carves the caller's workspace and enqueues
// kernels and NCCL calls on the caller's stream; every step of the path runs on
// the device (kernels.h).  One rank owns a z-slab of nzl = N/P planes (P = 1: the
// whole box).  One step:
//   SOLVE   fft_x_fwd -> fft_y_fwd -> [xpose] -> fft_z_mul -> [xpose] -> fft_y_inv
//           -> fft_x_inv (E4 + the halo plane of the slab below) -> energy (-> ncclAllReduce)
//   CLEAR   count = 0, rho = 0
//   PUSH    push_key (gather + kick + drift + key/rank; leavers -> their destination)
//           [P > 1: arrivals keyed]
//   SORT    scan -> place
//   SCATTER reorder_deposit (sorted gather + drift + stream out + CIC deposit; the charge
//           of node plane nzl goes to the next slab's plane 0)
// P > 1 has two transports.  Peer memory (default): every rank's workspace is mapped
// (CUDA IPC, NVLink); fft_x_inv writes the halo plane of the slab below, push_key stages
// the leavers and k_leaver_copy streams them into the destination's receive buffer, the
// ghost charge plane is pulled over NVLink by the slab above (k_add_plane after a
// barrier); the FFT transposes are copy-engine pulls of each peer's block after a barrier
// (ncclAlltoAll with PIC_XPOSE_PULL=0; the peer-store variant, PIC_P2P=2, measured
// slower).  NCCL (PIC_P2P=0 or no IPC): [xpose] = ncclAlltoAll, halo/ghost
// planes by ncclSend/Recv, leavers by counts all-to-all + grouped send/recv.
// Pencils (pgrid = {Py > 1, Pz}): a rank owns y and z blocks; the SOLVE is wrapped by a
// y-group redistribution of the charge to the FFT's z-slabs and one of the field back
// (pencil_to_slab_rho, slab_to_pencil_E: copy-engine pulls over the IPC mapping, else NCCL
// all-to-alls), and the ghost charge is folded in two phases (plane to +z, then row to +y:
// fold_ghost_pencil); migration, halos and ghost folds use NCCL.
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <vector>

#include "../../include/pic.h"
#include "kernels.h"

using pic::Geom;
using pic::PState;
using pic::SpecLayout;

namespace {

thread_local char g_init_error[512] = "";
constexpr int kMaxEnergySteps = 4096;   // device ring of per-step (W_x, W)

const char* kStageNames[PIC_NSTAGES] = {
    "fft_x_fwd", "fft_y_fwd", "fft_z_mul", "fft_y_inv", "fft_x_inv", "energy",
    "clear",     "push_key",  "scan",      "place",     "reorder_deposit", "exchange", "xpose",
    "pcg_ssor",  "pcg_cg",    "pcg_field"};

size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

bool is_pow2(int v) { return v > 0 && (v & (v - 1)) == 0; }

int ilog2i(int v) {
    int l = 0;
    while ((1 << l) < v) ++l;
    return l;
}

}  // namespace

struct pic_ctx {
    pic_params p{};
    Geom g{};                     // this rank's particle / real-space domain (slab or pencil)
    Geom gs{};                    // the FFT's z-slab geometry (== g for slabs, Py = 1)
    bool pencil = false;          // Py > 1: pencil domains; the solve redistributes to z-slabs
    int64_t np = 0;               // particles on this rank now
    int64_t np_cap = 0;           // capacity of the particle arrays of this rank
    int64_t np_glob = 0;          // N_p of the whole box
    int64_t ncell = 0;            // cells of the slab, n^2 nzl
    double q = 0.0;               // macro charge -L^3 / N_p
    double deposit_scale = 0.0;   // q inv_h^3 (raw CIC weight sums -> rho)
    cudaStream_t stream = nullptr;
    bool poisoned = false;
    char err[512] = "";
    double2* part[2][2] = {};     // double-buffered particle streams XY, ZV (pic_device.cuh)
    int cur = 0;
    uint32_t* key = nullptr;      // [np_cap + recv_cap] (extended index space)
    uint16_t* rank = nullptr;
    uint32_t* perm = nullptr;     // [np_cap]
    uint32_t* count = nullptr;
    uint32_t* offs = nullptr;
    uint32_t* bprev = nullptr;        // [nbrick + 1] brick ranges of the particle order push_key read
    uint32_t* scan_scratch = nullptr;
    double* rho = nullptr;        // (nzl + 1) pitched real planes; half spectrum S0 in the solve
    double2* specA = nullptr;     // forward transpose send (P = 1: rho)
    double2* specB = nullptr;     // ky-pencil (P = 1: rho)
    double2* specC = nullptr;     // 3 components: z-pass out, y-inverse out
    double2* specD = nullptr;     // return transpose receive (P = 1: specC)
    bool spec_alias = false;      // P = 1: specC/specD inside the idle particle buffer (bind_spec)
    size_t spec_unit = 0;
    double* E4 = nullptr;         // (nzl + 1) planes of node records (E_x, E_y, E_z, 0)
    double* ghost = nullptr;      // P > 1: received ghost plane of rho
    double2* tw = nullptr;
    double* partials = nullptr;
    double* energies = nullptr;   // ring [kMaxEnergySteps][2]
    int* err_flag = nullptr;
    int last_slot = -1;
    // migration (P > 1)
    double2* send = nullptr;      // [P][seg][4]
    uint32_t* send_count = nullptr;
    uint32_t* recv_count = nullptr;
    pic::SendSegs segs{};
    double2* recv = nullptr;      // [recv_cap][4]
    int64_t recv_cap = 0;
    int64_t migrated = 0;         // particles sent by this rank (all steps)
    ncclComm_t comm = nullptr;
    // pencils (Py > 1): the y-group communicator (the Py ranks sharing pz), the FFT's slab
    // buffers, and the staging buffers of the redistributions and ghost folds
    ncclComm_t ycomm = nullptr;
    double* rho_s = nullptr;      // slab S0 [nzs + 1][n][rp] (== rho for slabs)
    double* E4_s = nullptr;       // slab field [nzs + 1][n][n][4] (== E4 for slabs)
    double* xr[2] = {};           // rho pencil -> slab all-to-all: send, recv [Py][nzs][nyl][rp]
    double* xe[2] = {};           // E4 slab -> pencil all-to-all: send, recv [Py][nzs + 1][nyl + 1][n][4]
    double* fold[2] = {};         // ghost plane / row staging: send, recv (max(nyr rp, nzl rp) doubles)
    bool pen_alias = false;       // the pencil scratch in the idle particle buffer (bind_pencil)
    char* pen_own = nullptr;      // else its own space
    // peer-memory transport (P > 1): every rank's workspace mapped into this process
    // (CUDA IPC over NVLink); transposes, halo/ghost planes and migration are stores
    // and atomics of the producing kernels into the peers' buffers, ordered by
    // stream barriers (a one-int ncclAllReduce) instead of NCCL data movement
    bool p2p = false;
    bool xpose_p2p = false;               // transposes too (PIC_P2P=2; slower, see solve())
    bool ghost_p2p = false;               // ghost charge by peer atomics (else the NCCL fold)
    double2** peer_tab = nullptr;         // device [4][8]: every rank's specB, specD, specA, specC
    bool xpose_pull = false;              // transposes by peer pulls (PIC_XPOSE_PULL=1: kernel, 2: copy engines)
    bool xpose_ce = false;                // PIC_XPOSE_PULL=2
    bool xpose_split = false;             // PIC_XPOSE_SPLIT: pulls overlapped with the y / z pass halves
    bool ipc = false;                     // every rank's workspace mapped (peer_ws); p2p = ipc on z-slabs
    bool pen_ce = false;                  // pencils: y-group redistributions by copy-engine pulls
    bool mig_p2p = false;                 // particle migration through the peers' receive buffers
    cudaStream_t side[8] = {};            // copy-engine pulls, one stream per source rank
    cudaEvent_t side_ev[9] = {};
    char* ws = nullptr;                   // this rank's workspace base
    char* peer_ws[8] = {};                // rank r's workspace base in this address space
    void* ipc_open[8] = {};               // mapped peer allocations (closed by pic_free)
    int* bar = nullptr;                   // barrier word
    unsigned long long* dcnt = nullptr;   // device counts (pic::DC_*)
    bool np_stale = false;                // np / migrated live on the device (dcnt) until the next sync
    // FD-PCG solver (p.solver == PIC_SOLVER_PCG): colour-split fields of the slab
    double* pcg_x = nullptr;      // phi: the solution, kept as the next solve's warm start
    double* pcg_r = nullptr;
    double* pcg_z = nullptr;
    double* pcg_p[2] = {};        // search direction, ping-pong (the matvec forms p' = z + beta p)
    double* pcg_q = nullptr;      // A p
    double* pcg_sc = nullptr;     // device scalars (kernels.h)
    int pcg_pi = 0;
    int32_t pcg_last_iters = 0;
    int64_t pcg_total_iters = 0;
    int64_t pcg_solves = 0;
    int64_t pcg_launches = 0;     // kernel launches of the latest solve
    double pcg_last_relres = 0.0;
    // timing
    bool timing = false;
    double stage_ms[PIC_NSTAGES] = {};
    int64_t stage_launches[PIC_NSTAGES] = {};
    std::vector<cudaEvent_t> ev_pool;
    std::vector<int> ev_stage;
    size_t ev_used = 0;
};

namespace {

// ------------------------------------------------------------ validation ---
pic_status validate(const pic_params* p, int32_t rank, int32_t nranks, char* msg, size_t msz) {
    if (!p) { snprintf(msg, msz, "params is NULL"); return PIC_EINVAL; }
    if (!(nranks == 1 || nranks == 2 || nranks == 4 || nranks == 8) || rank < 0 || rank >= nranks) {
        snprintf(msg, msz, "nranks=%d rank=%d: nranks must be 1, 2, 4 or 8", nranks, rank);
        return PIC_EINVAL;
    }
    const int Py = p->pgrid[0], Pz = p->pgrid[1];
    if (!(Py >= 1 && Pz >= 1 && Py * Pz == nranks)) {
        snprintf(msg, msz, "pgrid = {%d, %d}: need Py * Pz == nranks = %d", Py, Pz, nranks);
        return PIC_EINVAL;
    }
    if (!is_pow2(p->n) || p->n < 16 || p->n > 1024) { snprintf(msg, msz, "n=%d: power of two in [16,1024]", p->n); return PIC_EINVAL; }
    if (p->n / nranks < 4) { snprintf(msg, msz, "n/nranks = %d: the FFT's z-slabs need >= 4 planes", p->n / nranks); return PIC_EINVAL; }
    if (Py > 1 && (p->n / Py < 8 || p->n / Pz < 4)) {
        snprintf(msg, msz, "pencils {%d, %d}: need n/Py >= 8 rows and n/Pz >= 4 planes", Py, Pz);
        return PIC_EINVAL;
    }
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
    if (p->solver != PIC_SOLVER_FFT && p->solver != PIC_SOLVER_PCG && p->solver != PIC_SOLVER_FEM) {
        snprintf(msg, msz, "solver=%d: PIC_SOLVER_FFT (0), PIC_SOLVER_PCG (1) or PIC_SOLVER_FEM (2)", p->solver);
        return PIC_EINVAL;
    }
    if (Py > 1 && p->solver != PIC_SOLVER_FFT) {
        snprintf(msg, msz, "pencils (pgrid = {%d, %d}) run the FFT solver only; PCG / FEM decompose in z-slabs", Py, Pz);
        return PIC_EUNSUPPORTED;
    }
    if (p->solver != PIC_SOLVER_FFT &&
        (!(p->pcg_tol > 0) || !(p->pcg_omega > 0 && p->pcg_omega < 2) || p->pcg_inner < 1 || p->pcg_outer < 1 ||
         p->pcg_maxit < 1)) {
        snprintf(msg, msz, "PCG: need tol > 0, 0 < omega < 2, inner >= 1, outer >= 1, maxit >= 1");
        return PIC_EINVAL;
    }
    for (int d = 0; d < 3; ++d)
        if (!std::isfinite(p->b_ext[d]) || !std::isfinite(p->e_ext[d])) {
            snprintf(msg, msz, "b_ext / e_ext must be finite");
            return PIC_EINVAL;
        }
    return PIC_OK;
}

// The FFT's z-slab geometry of a rank: nzs = n / P planes at z0 = rank nzs, every row.
Geom slab_geom(const Geom& g) {
    Geom s = g;
    s.Py = 1;
    s.nzl = g.n / g.P;
    s.mz = ilog2i(s.nzl);
    s.z0 = g.rank * s.nzl;
    s.nyl = g.n;
    s.my = ilog2i(g.n);
    s.y0 = 0;
    s.nyr = g.n;
    return s;
}

Geom make_geom(const pic_params* p, int rank, int nranks) {
    Geom g{};
    g.n = p->n;
    g.nmask = p->n - 1;
    g.px = (int)align_up((size_t)(p->n / 2 + 1), 8);
    g.rp = 2 * g.px;
    g.L = p->length == 0.0 ? 2.0 * M_PI / p->k : p->length;
    g.inv_h = (double)p->n / g.L;
    g.dt = p->dt;
    g.qm_dt = -1.0 * p->dt;     // q/m = -1
    g.P = nranks;
    g.rank = rank;
    g.Py = p->pgrid[0] > 0 ? p->pgrid[0] : 1;
    const int Pz = nranks / g.Py, py = rank % g.Py, pz = rank / g.Py;
    g.nzl = p->n / Pz;
    g.mz = ilog2i(g.nzl);
    g.z0 = pz * g.nzl;
    g.nyl = p->n / g.Py;
    g.my = ilog2i(g.nyl);
    g.y0 = py * g.nyl;
    g.nyr = g.Py > 1 ? g.nyl + 1 : p->n;
    // external fields (D#32): the coefficients in the oracle's order (oracle_boris_coeffs)
    g.eext = p->e_ext[0] != 0.0 || p->e_ext[1] != 0.0 || p->e_ext[2] != 0.0;
    g.boris = p->b_ext[0] != 0.0 || p->b_ext[1] != 0.0 || p->b_ext[2] != 0.0;
    g.hq = 0.5 * (-1.0 * p->dt);
    for (int d = 0; d < 3; ++d) {
        g.ee[d] = p->e_ext[d];
        g.bt[d] = g.hq * p->b_ext[d];
    }
    const double tt = (g.bt[0] * g.bt[0] + g.bt[1] * g.bt[1]) + g.bt[2] * g.bt[2];
    for (int d = 0; d < 3; ++d) g.bs[d] = (2.0 * g.bt[d]) / (1.0 + tt);
    return g;
}

struct Sizes {
    int pcg;
    int64_t np_nom, np_cap, recv_cap, nkey, send_len;
    pic::SendSegs segs;
};

Sizes sizes(const pic_params* p, const Geom& g) {
    Sizes s{};
    s.pcg = p->solver == PIC_SOLVER_PCG || p->solver == PIC_SOLVER_FEM;   // the CG vectors
    const int64_t npg = (int64_t)p->ppc * p->n * p->n * p->n;
    s.np_nom = npg / g.P;
    if (g.P == 1) {
        s.np_cap = s.np_nom;
        s.recv_cap = 0;
        s.send_len = 0;
    } else {
        // domain imbalance <= alpha per decomposed dimension (density (1 + alpha cos k z),
        // times (1 + alpha cos k y) for pencils), plus fluctuations
        // (the mean of 1 + alpha cos over a block of L / Py rows is at most
        // 1 + alpha sin(pi / Py) / (pi / Py))
        const double fy = g.Py > 1 ? 1.0 + p->alpha * std::sin(M_PI / g.Py) / (M_PI / g.Py) : 1.0;
        const double imb = (1.0 + p->alpha) * fy;
        s.np_cap = (int64_t)(s.np_nom * imb * 1.05) + 65536;
        // a slab of nzl planes loses ~ E[max(v_z, 0)] dt / (nzl h) per step to each z
        // neighbour (1.3% at 512^3 / 8 ranks): neighbour segments hold 4%
        // of the slab, the others (only reached by |v_z| dt > nzl h) 0.2%; at
        // 1024^3 / 8 ranks this keeps the rank's workspace at ~144 GiB
        const int nb = (int)std::min<int64_t>(s.np_cap, (int64_t)(0.04 * s.np_cap) + 4096);
        const int far = (int)std::min<int64_t>(nb, (int64_t)(0.002 * s.np_cap) + 4096);
        // face neighbours (one block index differs by one, periodic, the other equal): the
        // z neighbours of a slab, the four around a pencil; a particle reaches any other
        // rank (a pencil's diagonal neighbours included) only by crossing two faces in one
        // step, ~(1.3%)^2 of the particles at 512^3 / 8 ranks
        const int Py = g.Py, Pz = g.P / g.Py, py = g.rank % Py, pz = g.rank / Py;
        auto near1 = [](int a, int b, int m) { const int d = ((a - b) % m + m) % m; return d == 1 || d == m - 1; };
        int64_t off = 0, rc = 0;
        for (int r = 0; r < g.P; ++r) {
            const int ry = r % Py, rz = r / Py;
            const bool nbr = r != g.rank && ((ry == py && near1(rz, pz, Pz)) || (rz == pz && near1(ry, py, Py)));
            const int cap = r == g.rank ? 0 : (nbr ? nb : far);
            s.segs.off[r] = off;
            s.segs.cap[r] = cap;
            off += cap;
            rc += cap;          // the relation is symmetric: r sends this rank as much room
        }
        s.send_len = off;
        s.recv_cap = rc;
    }
    s.nkey = s.np_cap + s.recv_cap;
    return s;
}

// The arrays indexed with uint32 (key, rank, perm, offs; the old index packed in a
// leaver's record) span the extended index space nkey = capacity + receive buffer.
pic_status validate_sizes(const Sizes& z, char* msg, size_t msz) {
    if ((double)z.nkey >= 4294967295.0 || (double)z.np_cap >= 4294967295.0) {
        snprintf(msg, msz, "particle index space of a rank (capacity %lld + receive buffer %lld) too large "
                 "for 32-bit indices", (long long)z.np_cap, (long long)z.recv_cap);
        return PIC_EINVAL;
    }
    return PIC_OK;
}

// Pencils: the solve's slab S0 [nzs + 1][n][rp], slab field [nzs + 1][n][n][4] and the
// redistribution staging (xr: 2 x [Py][nzs][nyl][rp], xe: 2 x [Py][nzs + 1][nyl + 1][n][4]).
size_t pencil_scratch_bytes(const Geom& g) {
    const int nzs = g.n / g.P;
    return sizeof(double) * ((size_t)(nzs + 1) * g.n * g.rp + 4 * (size_t)(nzs + 1) * g.n * g.n +
                             2 * (size_t)g.nzl * g.nyl * g.rp + 2 * 4 * (size_t)g.Py * (nzs + 1) * (g.nyl + 1) * g.n);
}

// Point the pencil scratch (pencil_scratch_bytes) at its space: the idle particle buffer
// (cur ^ 1) when pen_alias, else the context's own.  Called before every use.
void bind_pencil(pic_ctx* c) {
    if (!c->pencil) return;
    const Geom& g = c->g;
    const int nzs = g.n / g.P;
    char* b = c->pen_alias ? reinterpret_cast<char*>(c->part[c->cur ^ 1][0]) : c->pen_own;
    auto take = [&](size_t doubles) {
        double* p = reinterpret_cast<double*>(b);
        b += align_up(sizeof(double) * doubles, 256);
        return p;
    };
    c->rho_s = take((size_t)(nzs + 1) * g.n * g.rp);
    c->E4_s = take(4 * (size_t)(nzs + 1) * g.n * g.n);
    c->xr[0] = take((size_t)g.nzl * g.nyl * g.rp);
    c->xr[1] = take((size_t)g.nzl * g.nyl * g.rp);
    c->xe[0] = take(4 * (size_t)g.Py * (nzs + 1) * (g.nyl + 1) * g.n);
    c->xe[1] = take(4 * (size_t)g.Py * (nzs + 1) * (g.nyl + 1) * g.n);
}

// P = 1 with spec_alias: point the spectral scratch at the particle buffer that does not
// hold the state (cur ^ 1).  Called before every use of specC / specD.
void bind_spec(pic_ctx* c) {
    if (!c->spec_alias) return;
    char* idle = reinterpret_cast<char*>(c->part[c->cur ^ 1][0]);
    c->specC = reinterpret_cast<double2*>(idle);
    c->specD = reinterpret_cast<double2*>(idle + c->spec_unit);
}

// Carve the workspace; returns the bytes needed (pointers set when c != nullptr).
size_t carve(pic_ctx* c, const Geom& g, const Sizes& z, char* base) {
    size_t off = 0;
    auto take = [&](size_t bytes) -> char* {
        off = align_up(off, 256);
        char* ptr = base ? base + off : nullptr;
        off += bytes;
        return ptr;
    };
    const Geom gs = slab_geom(g);                                       // the FFT's slab
    const bool pencil = g.Py > 1;
    const int64_t ncell = (int64_t)g.n * g.nyl * g.nzl;
    const size_t plane = sizeof(double) * (size_t)g.nyr * g.rp;        // one pitched real plane (domain)
    const size_t splane = sizeof(double) * (size_t)g.n * g.rp;         // one pitched real plane (slab)
    const size_t unit = sizeof(double2) * (size_t)gs.nzl * g.n * g.px;  // one slab half spectrum
    for (int b = 0; b < 2; ++b) {      // XY then ZV back to back (48 B x cap: also the SoA scratch)
        char* xy = take(sizeof(double2) * (size_t)z.np_cap);
        char* zv = take(2 * sizeof(double2) * (size_t)z.np_cap);
        if (c) {
            c->part[b][0] = reinterpret_cast<double2*>(xy);
            c->part[b][1] = reinterpret_cast<double2*>(zv);
        }
    }
    const int64_t nblk = g.P > 1 ? pic::sample_blocks(z.np_nom * g.P) : 0;   // init scratch
    char* k = take(sizeof(uint32_t) * (size_t)std::max(z.nkey, nblk));
    char* rk = take(sizeof(uint16_t) * (size_t)z.nkey);
    char* pm = take(sizeof(uint32_t) * (size_t)std::max(z.np_cap, nblk + 1));
    char* cn = take(sizeof(uint32_t) * (size_t)ncell);
    char* of = take(sizeof(uint32_t) * (size_t)(ncell + 1));
    char* bp = take(sizeof(uint32_t) * (size_t)(ncell / 256 + 1));
    char* ss = take(pic::scan_scratch_bytes(std::max(ncell, nblk)));
    char* rh = take(plane * (size_t)(g.nzl + 1));
    char* sA = g.P > 1 ? take(unit) : nullptr;
    char* sB = g.P > 1 ? take(unit) : nullptr;
    // P = 1: the three spectral components live in the idle particle buffer when it is
    // large enough (48 B x capacity >= 3 units; ppc >= 1 at N >= 32): the solve runs
    // between a reorder and the next push, when that buffer holds nothing.  Saves
    // 24 B per node (26 GB at 1024^3, which makes 1024^3 x 1 ppc fit one GPU).
    const bool spec_alias = g.P == 1 && 48 * (size_t)z.np_cap >= 3 * unit;
    char* sC = spec_alias ? nullptr : take(3 * unit);
    char* sD = g.P > 1 ? take(2 * unit) : nullptr;
    char* e4 = take(sizeof(double) * 4 * (size_t)g.n * g.nyr * (g.nzl + 1));
    char* gh = g.P > 1 ? take(plane) : nullptr;
    // pencils: the FFT's slab S0 and field and the redistribution staging live only inside
    // the solve, so they sit in the idle particle buffer when it is large enough (bind_pencil;
    // 16 GB of the 58 GB at 1024^3 x 8 / 8 ranks), else in their own space
    const size_t fo_b = sizeof(double) * (size_t)g.rp * std::max(g.nyr, g.nzl);
    const size_t pen_b = pencil_scratch_bytes(g);
    const bool pen_alias = pencil && 48 * (size_t)z.np_cap >= pen_b + 6 * 256;
    char* pen = pencil && !pen_alias ? take(pen_b + 6 * 256) : nullptr;
    char* fo0 = pencil ? take(fo_b) : nullptr;
    char* fo1 = pencil ? take(fo_b) : nullptr;
    char* tw = take(sizeof(double2) * (size_t)g.n);
    char* pa = take(sizeof(double) * 3 * (size_t)pic::energy_partials(g));
    char* en = take(sizeof(double) * 2 * kMaxEnergySteps);
    char* ef = take(sizeof(int) * 4);
    char* sd = g.P > 1 ? take(sizeof(double2) * 4 * (size_t)z.send_len) : nullptr;
    char* sc = take(sizeof(uint32_t) * 2 * 8);
    char* br = take(sizeof(int) * 4);
    char* pt = take(sizeof(double2*) * 32);
    char* dc = take(sizeof(unsigned long long) * 4);
    char* rv = g.P > 1 ? take(sizeof(double2) * 4 * (size_t)z.recv_cap) : nullptr;
    char* pv[6] = {};
    for (int k = 0; k < 6 && z.pcg; ++k) pv[k] = take(sizeof(double) * (size_t)ncell);
    char* psc = z.pcg ? take(sizeof(double) * 8) : nullptr;
    if (c) {
        c->pcg_x = reinterpret_cast<double*>(pv[0]);
        c->pcg_r = reinterpret_cast<double*>(pv[1]);
        c->pcg_z = reinterpret_cast<double*>(pv[2]);
        c->pcg_p[0] = reinterpret_cast<double*>(pv[3]);
        c->pcg_p[1] = reinterpret_cast<double*>(pv[4]);
        c->pcg_q = reinterpret_cast<double*>(pv[5]);
        c->pcg_sc = reinterpret_cast<double*>(psc);
        c->key = reinterpret_cast<uint32_t*>(k);
        c->rank = reinterpret_cast<uint16_t*>(rk);
        c->perm = reinterpret_cast<uint32_t*>(pm);
        c->count = reinterpret_cast<uint32_t*>(cn);
        c->offs = reinterpret_cast<uint32_t*>(of);
        c->bprev = reinterpret_cast<uint32_t*>(bp);
        c->scan_scratch = reinterpret_cast<uint32_t*>(ss);
        c->rho = reinterpret_cast<double*>(rh);
        c->specA = g.P > 1 ? reinterpret_cast<double2*>(sA) : reinterpret_cast<double2*>(rh);
        c->specB = g.P > 1 ? reinterpret_cast<double2*>(sB) : reinterpret_cast<double2*>(rh);
        (void)splane;
        c->spec_alias = spec_alias;
        c->spec_unit = unit;
        c->specC = reinterpret_cast<double2*>(sC);
        // P = 1: the z pass's two components go to units 1-2 of specC; the field y pass
        // reads each tile whole before writing units 0-2 over the same footprint
        c->specD = reinterpret_cast<double2*>(g.P > 1 ? sD : sC + unit);
        if (spec_alias) bind_spec(c);
        c->E4 = reinterpret_cast<double*>(e4);
        c->rho_s = reinterpret_cast<double*>(rh);
        c->E4_s = reinterpret_cast<double*>(e4);
        c->pen_alias = pen_alias;
        c->pen_own = pen;
        c->fold[0] = reinterpret_cast<double*>(fo0);
        c->fold[1] = reinterpret_cast<double*>(fo1);
        c->ghost = reinterpret_cast<double*>(gh);
        c->tw = reinterpret_cast<double2*>(tw);
        c->partials = reinterpret_cast<double*>(pa);
        c->energies = reinterpret_cast<double*>(en);
        c->err_flag = reinterpret_cast<int*>(ef);
        c->send = reinterpret_cast<double2*>(sd);
        c->send_count = reinterpret_cast<uint32_t*>(sc);
        c->bar = reinterpret_cast<int*>(br);
        c->peer_tab = reinterpret_cast<double2**>(pt);
        c->dcnt = reinterpret_cast<unsigned long long*>(dc);
        c->recv_count = reinterpret_cast<uint32_t*>(sc) + 8;
        c->segs = z.segs;
        c->recv = reinterpret_cast<double2*>(rv);
        c->recv_cap = z.recv_cap;
        c->np_cap = z.np_cap;
    }
    return align_up(off, 256);
}

pic_status fail(pic_ctx* c, pic_status st, const char* what, cudaError_t e = cudaSuccess) {
    if (e != cudaSuccess)
        snprintf(c->err, sizeof(c->err), "%s: %s", what, cudaGetErrorString(e));
    else
        snprintf(c->err, sizeof(c->err), "%s", what);
    if (st == PIC_ECUDA || st == PIC_ENCCL || st == PIC_EOVERFLOW) c->poisoned = true;
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

#define PIC_NCCL(ctx, call)                                                                     \
    do {                                                                                        \
        ncclResult_t r_ = (call);                                                               \
        if (r_ != ncclSuccess) {                                                                \
            snprintf((ctx)->err, sizeof((ctx)->err), "%s: %s", #call, ncclGetErrorString(r_)); \
            (ctx)->poisoned = true;                                                             \
            return PIC_ENCCL;                                                                   \
        }                                                                                       \
    } while (0)

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
    s.xy = c->part[b][0];
    s.zv = c->part[b][1];
    return s;
}

int up(const pic_ctx* c) { return (c->g.rank + 1) % c->g.P; }
int down(const pic_ctx* c) { return (c->g.rank + c->g.P - 1) % c->g.P; }

// The same workspace object on rank r (peer-memory transport; every rank carves an
// identical layout).
template <class T>
T* on_rank(const pic_ctx* c, int r, T* local) {
    return reinterpret_cast<T*>(c->peer_ws[r] + (reinterpret_cast<char*>(local) - c->ws));
}

// Stream barrier of all ranks: the peer stores/atomics of the kernels before it are
// complete (they end with a system fence) when any rank's work after it starts.
pic_status barrier(pic_ctx* c) {
    PIC_NCCL(c, ncclAllReduce(c->bar, c->bar, 1, ncclInt, ncclSum, c->comm, c->stream));
    return PIC_OK;
}

// A decision every rank must take together (a rank that bails out alone
// leaves its peers blocked in the next collective): 1 if any rank passes local != 0.
// Synchronises the stream.
pic_status agree_any(pic_ctx* c, int local, int* any) {
    *any = local;
    if (c->g.P == 1) return PIC_OK;
    int* d = c->bar + 2;
    PIC_CUDA(c, cudaMemcpyAsync(d, &local, sizeof(int), cudaMemcpyHostToDevice, c->stream));
    PIC_NCCL(c, ncclAllReduce(d, d, 1, ncclInt, ncclMax, c->comm, c->stream));
    PIC_CUDA(c, cudaMemcpyAsync(any, d, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    PIC_CUDA(c, cudaStreamSynchronize(c->stream));
    return PIC_OK;
}

// E halo plane nzl = the next slab's plane 0 (P = 1 and the peer-memory transport:
// written by fft_x_inv itself).
// The FFT's slab field: halo plane nzs = the next slab's plane 0 (slab order = rank order).
pic_status fill_E_halo(pic_ctx* c) {
    const Geom& g = c->gs;
    if (g.P == 1 || c->p2p) return PIC_OK;
    const size_t pl = (size_t)4 * g.n * g.n;   // doubles per E4 plane
    double* halo = c->E4_s + pl * g.nzl;
    PIC_NCCL(c, ncclGroupStart());
    PIC_NCCL(c, ncclSend(c->E4_s, pl, ncclDouble, down(c), c->comm, c->stream));
    PIC_NCCL(c, ncclRecv(halo, pl, ncclDouble, up(c), c->comm, c->stream));
    PIC_NCCL(c, ncclGroupEnd());
    return PIC_OK;
}

// ---------------------------------------------------------------- pencils ----
// Rank r = pz Py + py owns y in [py nyl, +nyl), z in [pz nzl, +nzl).  The FFT runs on z-slabs
// of nzs = n / P planes (slab index = rank): the Py ranks of a y-group (same pz) hold the same
// nzl planes, split in y, and their slabs are those planes split in z (py's slab: planes
// [py nzs, +nzs) of the group's block) -- so each direction is one all-to-all in the y-group.
int pen_rank(const pic_ctx* c, int py, int pz) {
    const int Py = c->g.Py, Pz = c->g.P / Py;
    return ((pz % Pz + Pz) % Pz) * Py + ((py % Py) + Py) % Py;
}

// rho of the pencil [nzl][nyl] -> the slab S0 [nzs][n] (rows y = qs nyl + yl from rank qs).
// Copy-engine pulls of the y-group redistributions (pen_ce): one 2D copy per group member
// on its own stream (staggered start), joined into the library stream.
template <class F>
pic_status group_pulls(pic_ctx* c, F copy) {
    const Geom& g = c->g;
    const int Py = g.Py, py = g.rank % Py;
    PIC_CUDA(c, cudaEventRecord(c->side_ev[8], c->stream));
    for (int i = 0; i < Py; ++i) {
        const int q = (py + i) % Py;
        PIC_CUDA(c, cudaStreamWaitEvent(c->side[i], c->side_ev[8], 0));
        PIC_TRY(copy(q, c->side[i]));
        PIC_CUDA(c, cudaEventRecord(c->side_ev[i], c->side[i]));
        PIC_CUDA(c, cudaStreamWaitEvent(c->stream, c->side_ev[i], 0));
    }
    return PIC_OK;
}

pic_status pencil_to_slab_rho(pic_ctx* c) {
    const Geom& g = c->g;
    const int nzs = c->gs.nzl, Py = g.Py;
    const size_t rp8 = sizeof(double) * g.rp;
    if (c->pen_ce) {     // after a barrier (every pencil's rho folded): my slab planes of each member's rows
        const int py = g.rank % Py, pz = g.rank / Py;
        PIC_TRY(barrier(c));
        return group_pulls(c, [&](int q, cudaStream_t s) -> pic_status {
            const double* src = on_rank(c, pen_rank(c, q, pz), c->rho) + (size_t)py * nzs * g.nyr * g.rp;
            PIC_CUDA(c, cudaMemcpy2DAsync(c->rho_s + (size_t)q * g.nyl * g.rp, (size_t)g.n * rp8, src,
                                          g.nyr * rp8, g.nyl * rp8, nzs, cudaMemcpyDeviceToDevice, s));
            return PIC_OK;
        });
    }
    const size_t blk = (size_t)nzs * g.nyl * g.rp;          // doubles per destination
    for (int q = 0; q < Py; ++q)       // planes [q nzs, +nzs), rows 0 .. nyl-1 of each (skip the ghost row)
        PIC_CUDA(c, cudaMemcpy2DAsync(c->xr[0] + q * blk, g.nyl * rp8, c->rho + (size_t)q * nzs * g.nyr * g.rp,
                                      g.nyr * rp8, g.nyl * rp8, nzs, cudaMemcpyDeviceToDevice, c->stream));
    PIC_NCCL(c, ncclAlltoAll(c->xr[0], c->xr[1], blk, ncclDouble, c->ycomm, c->stream));
    for (int q = 0; q < Py; ++q)       // from rank q of the group: its rows of my slab planes
        PIC_CUDA(c, cudaMemcpy2DAsync(c->rho_s + (size_t)q * g.nyl * g.rp, (size_t)g.n * rp8, c->xr[1] + q * blk,
                                      g.nyl * rp8, g.nyl * rp8, nzs, cudaMemcpyDeviceToDevice, c->stream));
    return PIC_OK;
}

// The slab field E4_s (planes 0 .. nzs, the last one its halo) -> the pencil E4 [nzl + 1][nyl + 1]:
// rank q of the group gets rows [q nyl, q nyl + nyl] (the last one wrapping) of the slab's
// nzs + 1 planes; the pencil's plane qs nzs + nzs comes twice (rank qs's halo, rank qs + 1's
// plane 0: the same values).
pic_status slab_to_pencil_E(pic_ctx* c) {
    const Geom& g = c->g;
    const int nzs = c->gs.nzl, Py = g.Py;
    if (c->pen_ce) {     // 32-B node records pulled as they are: no pack / unpack kernels
        const int py = g.rank % Py, pz = g.rank / Py;
        const size_t row8 = sizeof(double) * 4 * g.n;
        PIC_TRY(barrier(c));        // every slab field (and its halo plane) complete
        PIC_TRY(group_pulls(c, [&](int qs, cudaStream_t s) -> pic_status {
            const double* src = on_rank(c, pen_rank(c, qs, pz), c->E4_s);
            double* dst = c->E4 + (size_t)qs * nzs * g.nyr * 4 * g.n;
            PIC_CUDA(c, cudaMemcpy2DAsync(dst, g.nyr * row8, src + (size_t)py * g.nyl * 4 * g.n, g.n * row8,
                                          g.nyl * row8, nzs + 1, cudaMemcpyDeviceToDevice, s));
            const int yw = (py * g.nyl + g.nyl) & (g.n - 1);        // halo row nyl (wraps at the last py)
            PIC_CUDA(c, cudaMemcpy2DAsync(dst + (size_t)g.nyl * 4 * g.n, g.nyr * row8, src + (size_t)yw * 4 * g.n,
                                          g.n * row8, row8, nzs + 1, cudaMemcpyDeviceToDevice, s));
            return PIC_OK;
        }));
        return barrier(c);          // nobody overwrites its slab field (idle particle buffer) before all pulled
    }
    const size_t blk = (size_t)(nzs + 1) * (g.nyl + 1) * 3 * g.n;          // doubles per destination (24 B/node)
    pic::launch_e4_pencil_pack(c->E4_s, g.n, nzs, g.nyl, Py, c->xe[0], c->stream);
    PIC_LAUNCHED(c, "e4_pencil_pack");
    PIC_NCCL(c, ncclAlltoAll(c->xe[0], c->xe[1], blk, ncclDouble, c->ycomm, c->stream));
    pic::launch_e4_pencil_unpack(c->xe[1], g.n, nzs, g.nyl, Py, c->E4, c->stream);
    PIC_LAUNCHED(c, "e4_pencil_unpack");
    return PIC_OK;
}

// Ghost charge of a pencil (raw CIC sums on plane nzl and row nyl of the local grid) folded
// into the owners: the ghost plane (rows 0 .. nyl, i.e. with the edge) to the +z neighbour's
// plane 0, then the ghost row of planes 0 .. nzl-1 (the edge now included at plane 0 of the
// +z neighbour) to the +y neighbour's row 0.
pic_status fold_ghost_pencil(pic_ctx* c) {
    const Geom& g = c->g;
    const int Py = g.Py, py = g.rank % Py, pz = g.rank / Py;
    const int64_t plane = (int64_t)g.nyr * g.rp;
    PIC_NCCL(c, ncclGroupStart());
    PIC_NCCL(c, ncclSend(c->rho + plane * g.nzl, (size_t)plane, ncclDouble, pen_rank(c, py, pz + 1), c->comm, c->stream));
    PIC_NCCL(c, ncclRecv(c->fold[1], (size_t)plane, ncclDouble, pen_rank(c, py, pz - 1), c->comm, c->stream));
    PIC_NCCL(c, ncclGroupEnd());
    pic::launch_add_plane(c->rho, c->fold[1], plane, c->stream);
    PIC_LAUNCHED(c, "add_plane");
    const size_t rp8 = sizeof(double) * g.rp;
    PIC_CUDA(c, cudaMemcpy2DAsync(c->fold[0], rp8, c->rho + (size_t)g.nyl * g.rp, plane * sizeof(double), rp8,
                                  g.nzl, cudaMemcpyDeviceToDevice, c->stream));
    PIC_NCCL(c, ncclGroupStart());
    PIC_NCCL(c, ncclSend(c->fold[0], (size_t)g.nzl * g.rp, ncclDouble, pen_rank(c, py + 1, pz), c->comm, c->stream));
    PIC_NCCL(c, ncclRecv(c->fold[1], (size_t)g.nzl * g.rp, ncclDouble, pen_rank(c, py - 1, pz), c->comm, c->stream));
    PIC_NCCL(c, ncclGroupEnd());
    pic::launch_add_rows(c->rho, plane, c->fold[1], g.rp, g.rp, g.nzl, c->stream);
    PIC_LAUNCHED(c, "add_rows");
    return PIC_OK;
}

// Halo row and plane of a pencil's E4 written outside the solve (pic_push_injected): the
// halo row of planes 0 .. nzl-1 from the +y neighbour's row 0, then the halo plane (rows
// 0 .. nyl: with the edge) from the +z neighbour's plane 0.
pic_status halo_pencil(pic_ctx* c) {
    const Geom& g = c->g;
    bind_pencil(c);
    const int Py = g.Py, py = g.rank % Py, pz = g.rank / Py;
    const size_t row = (size_t)4 * g.n, plane = row * g.nyr;            // doubles
    double* tmp0 = c->xe[0];
    double* tmp1 = c->xe[1];
    PIC_CUDA(c, cudaMemcpy2DAsync(tmp0, row * sizeof(double), c->E4, plane * sizeof(double), row * sizeof(double),
                                  g.nzl, cudaMemcpyDeviceToDevice, c->stream));
    PIC_NCCL(c, ncclGroupStart());
    PIC_NCCL(c, ncclSend(tmp0, row * g.nzl, ncclDouble, pen_rank(c, py - 1, pz), c->comm, c->stream));
    PIC_NCCL(c, ncclRecv(tmp1, row * g.nzl, ncclDouble, pen_rank(c, py + 1, pz), c->comm, c->stream));
    PIC_NCCL(c, ncclGroupEnd());
    PIC_CUDA(c, cudaMemcpy2DAsync(c->E4 + row * g.nyl, plane * sizeof(double), tmp1, row * sizeof(double),
                                  row * sizeof(double), g.nzl, cudaMemcpyDeviceToDevice, c->stream));
    PIC_NCCL(c, ncclGroupStart());
    PIC_NCCL(c, ncclSend(c->E4, plane, ncclDouble, pen_rank(c, py, pz - 1), c->comm, c->stream));
    PIC_NCCL(c, ncclRecv(c->E4 + plane * g.nzl, plane, ncclDouble, pen_rank(c, py, pz + 1), c->comm, c->stream));
    PIC_NCCL(c, ncclGroupEnd());
    return PIC_OK;
}

// Halo plane of a field written outside the solve (pic_push_injected).
pic_status refresh_halo(pic_ctx* c) {
    const Geom& g = c->g;
    if (c->pencil) return halo_pencil(c);
    const size_t pl = (size_t)4 * g.n * g.n;
    double* halo = c->E4 + pl * g.nzl;
    if (g.P == 1) {
        PIC_CUDA(c, cudaMemcpyAsync(halo, c->E4, sizeof(double) * pl, cudaMemcpyDeviceToDevice, c->stream));
        return PIC_OK;
    }
    if (!c->p2p) return fill_E_halo(c);
    PIC_TRY(barrier(c));     // the rank above has written its plane 0
    PIC_CUDA(c, cudaMemcpyAsync(halo, on_rank(c, up(c), c->E4), sizeof(double) * pl, cudaMemcpyDeviceToDevice,
                                c->stream));
    return barrier(c);
}

// Peer-pull transpose (after a barrier: every send side complete): block rank of rank q's
// send buffer src -> block q of dst, blk complex elements per block.  PIC_XPOSE_PULL=1: one
// kernel reads all peers over NVLink; 2: one copy-engine memcpy per source rank, each on
// its own stream (staggered start, so that the ranks do not all read one peer at once).
pic_status xpose_pull(pic_ctx* c, double2* dst, double2* src, double2* const* src_tab, int64_t blk) {
    const Geom& g = c->gs;
    if (!c->xpose_ce) {
        pic::launch_xpose_pull(dst, src_tab, blk, g.rank, g.P, c->stream);
        PIC_LAUNCHED(c, "xpose_pull");
        return PIC_OK;
    }
    PIC_CUDA(c, cudaEventRecord(c->side_ev[8], c->stream));
    for (int i = 0; i < g.P; ++i) {
        const int q = (g.rank + i) % g.P;
        const double2* from = (q == g.rank ? src : on_rank(c, q, src)) + (size_t)g.rank * blk;
        PIC_CUDA(c, cudaStreamWaitEvent(c->side[i], c->side_ev[8], 0));
        PIC_CUDA(c, cudaMemcpyAsync(dst + (size_t)q * blk, from, sizeof(double2) * (size_t)blk,
                                    cudaMemcpyDeviceToDevice, c->side[i]));
        PIC_CUDA(c, cudaEventRecord(c->side_ev[i], c->side[i]));
        PIC_CUDA(c, cudaStreamWaitEvent(c->stream, c->side_ev[i], 0));
    }
    return PIC_OK;
}

// One part of every transpose block by copy-engine pulls: dst block q + off <- rank q's src
// block rank + off, width bytes x height rows at pitch bytes, forked from the library stream
// (join: the library stream waits for all of them).
pic_status xpose_part(pic_ctx* c, double2* dst, double2* src, int64_t blk, int64_t off, size_t width,
                      size_t height, size_t pitch, bool join) {
    const Geom& g = c->gs;
    PIC_CUDA(c, cudaEventRecord(c->side_ev[8], c->stream));
    for (int i = 0; i < g.P; ++i) {
        const int q = (g.rank + i) % g.P;
        const double2* from = (q == g.rank ? src : on_rank(c, q, src)) + (size_t)g.rank * blk + off;
        PIC_CUDA(c, cudaStreamWaitEvent(c->side[i], c->side_ev[8], 0));
        PIC_CUDA(c, cudaMemcpy2DAsync(dst + (size_t)q * blk + off, pitch, from, pitch, width, height,
                                      cudaMemcpyDeviceToDevice, c->side[i]));
        if (join) {
            PIC_CUDA(c, cudaEventRecord(c->side_ev[i], c->side[i]));
            PIC_CUDA(c, cudaStreamWaitEvent(c->stream, c->side_ev[i], 0));
        }
    }
    return PIC_OK;
}

// The split transposes (PIC_XPOSE_SPLIT; pencils by default): both halves non-empty.
bool xpose_split(const pic_ctx* c) {
    return c->gs.P > 1 && c->xpose_ce && c->xpose_split && c->gs.nzl >= 2;
}

// Destination of fft_x_inv's copy of plane 0: the halo plane of the slab below.
double* halo_dst(pic_ctx* c) {
    const Geom& g = c->gs;
    double* own = c->E4_s + (size_t)4 * g.n * g.n * g.nzl;
    if (g.P == 1) return own;
    return c->p2p ? on_rank(c, down(c), own) : nullptr;
}

// Destination of reorder_deposit's charge on node plane nzl (plane 0 of the next slab).
double* ghost_dst(pic_ctx* c) {
    const Geom& g = c->g;
    if (g.P == 1) return c->rho;
    if (c->ghost_p2p) return on_rank(c, up(c), c->rho);   // PIC_P2P_GHOST=2 (slower, see below)
    return c->rho + (int64_t)g.nyr * g.rp * g.nzl;
}

// NCCL transport: rho ghost plane nzl (charge of the next slab's plane 0) folded into its owner.
// Peer transport: after a barrier, each rank pulls the ghost plane of the slab below
// over NVLink (coalesced 16-B loads) and adds it to its plane 0.  Adding it from the
// producer with system-scope RED.ADD.F64 inside reorder_deposit (PIC_P2P_GHOST=2) was
// measured 2.6 ms slower at 512^3 / 2 ranks.
pic_status fold_rho_ghost(pic_ctx* c) {
    const Geom& g = c->g;
    if (g.P == 1 || c->ghost_p2p) return PIC_OK;
    if (c->pencil) return fold_ghost_pencil(c);
    const int64_t pl = (int64_t)g.n * g.rp;
    double* ghost = c->rho + pl * g.nzl;
    if (c->p2p) {
        PIC_TRY(barrier(c));
        pic::launch_add_plane(c->rho, on_rank(c, down(c), ghost), pl, c->stream);
        PIC_LAUNCHED(c, "add_plane");
        return PIC_OK;
    }
    PIC_NCCL(c, ncclGroupStart());
    PIC_NCCL(c, ncclSend(ghost, (size_t)pl, ncclDouble, up(c), c->comm, c->stream));
    PIC_NCCL(c, ncclRecv(c->ghost, (size_t)pl, ncclDouble, down(c), c->comm, c->stream));
    PIC_NCCL(c, ncclGroupEnd());
    pic::launch_add_plane(c->rho, c->ghost, pl, c->stream);
    PIC_LAUNCHED(c, "add_plane");
    return PIC_OK;
}

// rho (raw CIC sums of the slab, scaled by `scale` in the multiply) -> E4 with its
// halo plane, energies (summed over ranks) -> ring slot.
pic_status solve(pic_ctx* c, double scale, int slot) {
    const Geom& g = c->gs;            // the FFT runs on z-slabs (pencils: redistributed first)
    bind_spec(c);
    bind_pencil(c);
    if (c->pencil) {
        StageScope t(c, PIC_STAGE_XPOSE, 0);
        PIC_TRY(pencil_to_slab_rho(c));
    }
    const size_t unit = (size_t)g.nzl * g.n * g.px;   // complex per slab half spectrum
    const SpecLayout S0{reinterpret_cast<double2*>(c->rho_s), 0, 1, nullptr};
    SpecLayout A{c->specA, 1, 1, nullptr};          // forward transpose, send side
    SpecLayout Cz{g.P > 1 ? c->specC : c->specD, 1, 2, nullptr};   // return transpose, send side
    const SpecLayout D{c->specD, 1, 2, nullptr};
    const SpecLayout C{c->specC, 0, 3, nullptr};
    // Transposes: copy-engine pulls on the peer transport (xpose_pull), else NCCL all-to-alls.
    // Storing the 64-byte column runs of the y/z passes straight into the peers (SpecLayout
    // REMOTE, PIC_P2P=2) was measured slower at P = 2 (z pass 0.95 -> 2.6 ms).
    const bool xpose_p2p = c->p2p && c->xpose_p2p;
    if (xpose_p2p) {
        A.packed = Cz.packed = 2;
        A.peer = c->peer_tab;
        Cz.peer = c->peer_tab + 8;
    }
    { StageScope t(c, PIC_STAGE_FFT_X_FWD, 1); pic::launch_fft_x_fwd(g, c->rho_s, c->tw, c->stream); }
    PIC_LAUNCHED(c, "fft_x_fwd");
    if (xpose_split(c)) {
        // copy-engine transposes overlapped with the passes that produce them: the y pass in two
        // plane halves (the first half's blocks are pulled while the second is transformed),
        // the z pass in two ky-row halves likewise
        const int64_t pt = pic::fft_plane_tiles(g.n), zt = pic::fft_zrow_tiles(g.n);
        const int h = g.nzl / 2, nz = g.nzl;                    // nyl = nzl on the FFT's slabs
        const int64_t blkA = (int64_t)(unit / g.P), blkC = 2 * blkA;
        const size_t row = sizeof(double2) * (size_t)g.px;
        { StageScope t(c, PIC_STAGE_FFT_Y_FWD, 1); pic::launch_fft_y(g, S0, A, 1, 0, c->tw, c->stream, 0, h * pt); }
        PIC_LAUNCHED(c, "fft_y_fwd");
        {
            StageScope t(c, PIC_STAGE_XPOSE, 0);
            PIC_TRY(barrier(c));
            PIC_TRY(xpose_part(c, c->specB, c->specA, blkA, 0, h * nz * row, 1, h * nz * row, false));
        }
        { StageScope t(c, PIC_STAGE_FFT_Y_FWD, 1); pic::launch_fft_y(g, S0, A, 1, 0, c->tw, c->stream, h * pt, nz * pt); }
        PIC_LAUNCHED(c, "fft_y_fwd");
        {
            StageScope t(c, PIC_STAGE_XPOSE, 0);
            PIC_TRY(barrier(c));
            PIC_TRY(xpose_part(c, c->specB, c->specA, blkA, (int64_t)h * nz * g.px, (nz - h) * nz * row, 1,
                               (nz - h) * nz * row, true));
        }
        { StageScope t(c, PIC_STAGE_FFT_Z_MUL, 1); pic::launch_fft_z_mul(g, c->specB, Cz, scale, c->tw, c->stream, 0, h * zt); }
        PIC_LAUNCHED(c, "fft_z_mul");
        {
            StageScope t(c, PIC_STAGE_XPOSE, 0);
            PIC_TRY(barrier(c));
            PIC_TRY(xpose_part(c, c->specD, c->specC, blkC, 0, h * row, 2 * nz, nz * row, false));
        }
        {
            StageScope t(c, PIC_STAGE_FFT_Z_MUL, 1);
            pic::launch_fft_z_mul(g, c->specB, Cz, scale, c->tw, c->stream, h * zt, nz * zt);
        }
        PIC_LAUNCHED(c, "fft_z_mul");
        {
            StageScope t(c, PIC_STAGE_XPOSE, 0);
            PIC_TRY(barrier(c));
            PIC_TRY(xpose_part(c, c->specD, c->specC, blkC, (int64_t)h * g.px, (nz - h) * row, 2 * nz, nz * row, true));
            PIC_TRY(barrier(c));             // every rank has pulled from my specC before the field y pass
        }
    } else {
    { StageScope t(c, PIC_STAGE_FFT_Y_FWD, 1); pic::launch_fft_y(g, S0, A, 1, 0, c->tw, c->stream); }
    PIC_LAUNCHED(c, "fft_y_fwd");
    if (g.P > 1) {
        StageScope t(c, PIC_STAGE_XPOSE, 0);
        if (xpose_p2p) {
            PIC_TRY(barrier(c));
        } else if (c->xpose_pull) {          // every send buffer complete, then pull my blocks
            PIC_TRY(barrier(c));
            PIC_TRY(xpose_pull(c, c->specB, c->specA, c->peer_tab + 16, (int64_t)(unit / g.P)));
        } else {
            PIC_NCCL(c, ncclAlltoAll(c->specA, c->specB, 2 * unit / g.P, ncclDouble, c->comm, c->stream));
        }
    }
    { StageScope t(c, PIC_STAGE_FFT_Z_MUL, 1); pic::launch_fft_z_mul(g, c->specB, Cz, scale, c->tw, c->stream); }
    PIC_LAUNCHED(c, "fft_z_mul");
    if (g.P > 1) {
        StageScope t(c, PIC_STAGE_XPOSE, 0);
        if (xpose_p2p) {
            PIC_TRY(barrier(c));
        } else if (c->xpose_pull) {          // pull, then wait until every rank has pulled from my specC
            PIC_TRY(barrier(c));             // before the field y pass overwrites it
            PIC_TRY(xpose_pull(c, c->specD, c->specC, c->peer_tab + 24, (int64_t)(2 * unit / g.P)));
            PIC_TRY(barrier(c));
        } else {
            PIC_NCCL(c, ncclAlltoAll(c->specC, c->specD, 4 * unit / g.P, ncclDouble, c->comm, c->stream));
        }
    }
    }
    { StageScope t(c, PIC_STAGE_FFT_Y_INV, 1); pic::launch_fft_y_field(g, D, C, c->tw, c->stream); }
    PIC_LAUNCHED(c, "fft_y_inv");
    {
        StageScope t(c, PIC_STAGE_FFT_X_INV, 1);
        pic::launch_fft_x_inv(g, c->specC, c->E4_s, halo_dst(c), c->tw, c->partials, c->stream);
    }
    PIC_LAUNCHED(c, "fft_x_inv");
    { StageScope t(c, PIC_STAGE_ENERGY, 1); pic::launch_energy_reduce(g, c->partials, c->energies + 2 * slot, c->stream); }
    PIC_LAUNCHED(c, "energy");
    if (g.P > 1) {       // the energy sum is also the barrier for the halo stores
        StageScope t(c, PIC_STAGE_EXCHANGE, 0);
        PIC_NCCL(c, ncclAllReduce(c->energies + 2 * slot, c->energies + 2 * slot, 2, ncclDouble, ncclSum,
                                  c->comm, c->stream));
        PIC_TRY(fill_E_halo(c));
    }
    if (c->pencil) {
        StageScope t(c, PIC_STAGE_XPOSE, 0);
        PIC_TRY(slab_to_pencil_E(c));
    }
    c->last_slot = slot;
    return PIC_OK;
}

// ------------------------------------------------------------- FD-PCG -------
// A field of the slab with its neighbours' copies (planes -1 and nzl, kernels.h).
pic::PcgNbr pcg_nbr(pic_ctx* c, double* f) {
    if (c->g.P == 1) return pic::PcgNbr{f, f, f};
    return pic::PcgNbr{f, on_rank(c, down(c), f), on_rank(c, up(c), f)};
}

pic_status pcg_allreduce(pic_ctx* c, double* v, int n) {
    if (c->g.P > 1) PIC_NCCL(c, ncclAllReduce(v, v, n, ncclDouble, ncclSum, c->comm, c->stream));
    return PIC_OK;
}

pic_status pcg_read(pic_ctx* c, double* host, const double* dev, int n) {
    PIC_CUDA(c, cudaMemcpyAsync(host, dev, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
    PIC_CUDA(c, cudaStreamSynchronize(c->stream));
    return PIC_OK;
}

// z = M^-1 r (D#28): outer x {inner x (red, black), inner x (black, red)} SOR
// half-sweeps from z = 0; the last one also leaves (r, z) in sc[3] (old value in sc[4]).
// Default: one kernel per half-sweep, in place (k_sor).  PIC_PCG_TB=1: temporally
// blocked passes of pcg_tb_stages() half-sweeps (k_ssor_tb), ping-ponging between
// pcg_z and pcg_q (q is free between the update and the next matvec) so that the
// last pass lands in pcg_z -- a quarter of the HBM traffic, but measured slower
// (issue-bound: halo recomputation, ring addressing, a barrier per half-sweep).  P > 1: a barrier before every launch that reads
// what the peers wrote in the previous one.
pic_status pcg_precondition(pic_ctx* c) {
    const Geom& g = c->g;
    const int inner = c->p.pcg_inner, outer = c->p.pcg_outer;
    const int total = 4 * inner * outer;
    std::vector<int> colour;
    for (int o = 0; o < outer; ++o) {
        for (int i = 0; i < inner; ++i) { colour.push_back(0); colour.push_back(1); }
        for (int i = 0; i < inner; ++i) { colour.push_back(1); colour.push_back(0); }
    }
    const char* tbenv = getenv("PIC_PCG_TB");
    if (tbenv && tbenv[0] == '1') {
        const int T = pic::pcg_tb_stages();
        const int npass = (total + T - 1) / T;
        for (int k = 0; k < npass; ++k) {
            const int first = k * T, ns = std::min(T, total - first);
            int seq = 0;
            for (int t = 0; t < ns; ++t) seq |= colour[first + t] << t;
            const bool dot = k == npass - 1;
            double* zout = ((npass - 1 - k) % 2 == 0) ? c->pcg_z : c->pcg_q;
            double* zin = zout == c->pcg_z ? c->pcg_q : c->pcg_z;
            if (g.P > 1 && k > 0) PIC_TRY(barrier(c));
            StageScope t(c, PIC_STAGE_PCG_SSOR, dot ? 2 : 1);
            pic::launch_pcg_ssor_pass(g, ns, seq, k == 0, dot, pcg_nbr(c, c->pcg_r), pcg_nbr(c, zin), zout,
                                      c->p.pcg_omega, c->partials, c->pcg_sc, c->stream);
            PIC_LAUNCHED(c, "pcg_ssor_pass");
            c->pcg_launches += dot ? 2 : 1;
            if (dot) PIC_TRY(pcg_allreduce(c, c->pcg_sc + 3, 1));
        }
        return PIC_OK;
    }
    for (int k = 0; k < total; ++k) {
        const int mode = k == 0 ? 2 : (k == 1 ? 1 : 0);
        const bool dot = k == total - 1;
        if (g.P > 1 && mode != 2) PIC_TRY(barrier(c));
        StageScope t(c, PIC_STAGE_PCG_SSOR, dot ? 2 : 1);
        pic::launch_pcg_sor(g, colour[k], mode, dot, c->pcg_r, pcg_nbr(c, c->pcg_z), c->p.pcg_omega, c->partials,
                            c->pcg_sc, c->stream);
        PIC_LAUNCHED(c, "pcg_sor");
        c->pcg_launches += dot ? 2 : 1;
        if (dot) PIC_TRY(pcg_allreduce(c, c->pcg_sc + 3, 1));
    }
    return PIC_OK;
}

// The PCG solve (BJ config 5; D#26-D#31): rho = dscale * raw,
// b = rho - mean(rho), -Delta_h phi = b by SSOR-PCG warm-started from pcg_x, then
// E = -grad_h phi -> E4 (+ the halo plane of the slab below) and the energies.  The
// host reads (r, r) after every update (one stream synchronisation per iteration) to
// stop at ||r||^2 <= tol^2 ||b||^2.
pic_status solve_pcg(pic_ctx* c, double dscale, int slot) {
    const Geom& g = c->g;
    double* sc = c->pcg_sc;
    const double nn = (double)g.n * g.n * g.n;
    const double tol = c->p.pcg_tol;
    c->pcg_launches = 0;
    if (g.P > 1) PIC_TRY(barrier(c));          // the warm start x of every slab is in place
    {
        StageScope t(c, PIC_STAGE_PCG_CG, 4);
        pic::launch_pcg_rho_sum(g, c->rho, dscale, c->partials, sc, c->stream);
        PIC_LAUNCHED(c, "pcg_rho_sum");
        PIC_TRY(pcg_allreduce(c, sc, 1));
        pic::launch_pcg_resid0(g, c->rho, dscale, sc, nn, pcg_nbr(c, c->pcg_x), c->pcg_r, c->partials, c->stream);
        PIC_LAUNCHED(c, "pcg_resid0");
        PIC_TRY(pcg_allreduce(c, sc + 1, 2));
        c->pcg_launches += 4;
    }
    double h[3];
    PIC_TRY(pcg_read(c, h, sc + 1, 2));
    const double bb = h[0], stop = (tol * tol) * bb;
    double rr = h[1];
    int it = 0;
    bool converged = false;
    if (bb == 0.0) {
        PIC_CUDA(c, cudaMemsetAsync(c->pcg_x, 0, sizeof(double) * (size_t)c->ncell, c->stream));
        converged = true;
        rr = 0.0;
    } else if (rr <= stop) {
        converged = true;
    } else {
        PIC_TRY(pcg_precondition(c));                          // z = M^-1 r, sc[3] = (r, z)
        for (it = 1; it <= c->p.pcg_maxit; ++it) {
            const bool first = it == 1;
            double* pold = c->pcg_p[c->pcg_pi];
            double* pnew = c->pcg_p[c->pcg_pi ^ 1];
            {
                StageScope t(c, PIC_STAGE_PCG_CG, 4);
                pic::launch_pcg_matvec(g, first, pcg_nbr(c, c->pcg_z), pcg_nbr(c, pold), pnew, c->pcg_q, sc,
                                       c->partials, c->stream);    // p = z + beta p, q = A p, sc[5]
                PIC_LAUNCHED(c, "pcg_matvec");
                PIC_TRY(pcg_allreduce(c, sc + 5, 1));
                pic::launch_pcg_update(g, c->pcg_x, pnew, c->pcg_r, c->pcg_q, sc, c->partials, c->stream);
                PIC_LAUNCHED(c, "pcg_update");
                PIC_TRY(pcg_allreduce(c, sc + 2, 1));
                c->pcg_launches += 4;
            }
            c->pcg_pi ^= 1;
            PIC_TRY(pcg_read(c, &rr, sc + 2, 1));
            if (rr <= stop) { converged = true; break; }
            PIC_TRY(pcg_precondition(c));                      // z = M^-1 r, sc[3] = (r, z), sc[4] old
        }
    }
    c->pcg_last_iters = converged ? it : -1;
    c->pcg_total_iters += it > c->p.pcg_maxit ? c->p.pcg_maxit : it;
    c->pcg_solves += 1;
    c->pcg_last_relres = bb > 0.0 ? std::sqrt(rr / bb) : 0.0;
    {
        StageScope t(c, PIC_STAGE_PCG_FIELD, 2);
        pic::launch_pcg_gradient(g, pcg_nbr(c, c->pcg_x), c->E4, halo_dst(c), c->partials, c->energies + 2 * slot,
                                 c->stream);
        PIC_LAUNCHED(c, "pcg_gradient");
        c->pcg_launches += 2;
    }
    if (g.P > 1) {       // the energy sum is also the barrier for the halo stores
        StageScope t(c, PIC_STAGE_EXCHANGE, 0);
        PIC_NCCL(c, ncclAllReduce(c->energies + 2 * slot, c->energies + 2 * slot, 2, ncclDouble, ncclSum,
                                  c->comm, c->stream));
    }
    c->last_slot = slot;
    if (!converged) {
        snprintf(c->err, sizeof(c->err), "PCG did not converge in %d iterations (relative residual %.3e)",
                 c->p.pcg_maxit, c->pcg_last_relres);
        return PIC_ENONCONV;
    }
    return PIC_OK;
}

// The FEM solve (D#33): load
// b = h^3 dscale raw - mean, plain CG on the 27-point Q1 stiffness warm-started from
// pcg_x (natural layout), E = -grad_h phi -> E4 (+ the halo plane of the slab below).
pic_status solve_fem(pic_ctx* c, double dscale, int slot) {
    const Geom& g = c->g;
    double* sc = c->pcg_sc;
    const double nn = (double)g.n * g.n * g.n;
    const double tol = c->p.pcg_tol;
    c->pcg_launches = 0;
    if (g.P > 1) PIC_TRY(barrier(c));
    {
        StageScope t(c, PIC_STAGE_PCG_CG, 4);
        pic::launch_fem_load_sum(g, c->rho, dscale, c->partials, sc, c->stream);
        PIC_LAUNCHED(c, "fem_load_sum");
        PIC_TRY(pcg_allreduce(c, sc, 1));
        pic::launch_fem_resid0(g, c->rho, dscale, sc, nn, pcg_nbr(c, c->pcg_x), c->pcg_r, c->partials, c->stream);
        PIC_LAUNCHED(c, "fem_resid0");
        PIC_TRY(pcg_allreduce(c, sc + 1, 2));
        c->pcg_launches += 4;
    }
    double h[2];
    PIC_TRY(pcg_read(c, h, sc + 1, 2));
    const double bb = h[0], stop = (tol * tol) * bb;
    double rr = h[1];
    int it = 0;
    bool converged = false;
    if (bb == 0.0) {
        PIC_CUDA(c, cudaMemsetAsync(c->pcg_x, 0, sizeof(double) * (size_t)c->ncell, c->stream));
        converged = true;
        rr = 0.0;
    } else if (rr <= stop) {
        converged = true;
    } else {
        for (it = 1; it <= c->p.pcg_maxit; ++it) {
            double* pold = c->pcg_p[c->pcg_pi];
            double* pnew = c->pcg_p[c->pcg_pi ^ 1];
            StageScope t(c, PIC_STAGE_PCG_CG, 4);
            if (it > 1 && pic::fem_split()) {                  // p = r + beta p; q = A p, sc[5]
                pic::launch_fem_paxpy(g, c->pcg_r, pold, pnew, sc, c->stream);
                PIC_LAUNCHED(c, "fem_paxpy");
                if (g.P > 1) PIC_TRY(barrier(c));              // the peers' p is complete
                pic::launch_fem_stencil(g, pcg_nbr(c, pnew), c->pcg_q, sc, c->partials, c->stream);
                c->pcg_launches += 1;
            } else {
                pic::launch_fem_matvec(g, it == 1, pcg_nbr(c, c->pcg_r), pcg_nbr(c, pold), pnew, c->pcg_q, sc,
                                       c->partials, c->stream);      // p = r + beta p, q = A p, sc[5]
            }
            PIC_LAUNCHED(c, "fem_matvec");
            PIC_TRY(pcg_allreduce(c, sc + 5, 1));
            pic::launch_fem_update(g, c->pcg_x, pnew, c->pcg_r, c->pcg_q, sc, c->partials, c->stream);
            PIC_LAUNCHED(c, "fem_update");
            PIC_TRY(pcg_allreduce(c, sc + 2, 1));
            c->pcg_launches += 4;
            c->pcg_pi ^= 1;
            PIC_TRY(pcg_read(c, &rr, sc + 2, 1));
            if (rr <= stop) { converged = true; break; }
        }
    }
    c->pcg_last_iters = converged ? it : -1;
    c->pcg_total_iters += it > c->p.pcg_maxit ? c->p.pcg_maxit : it;
    c->pcg_solves += 1;
    c->pcg_last_relres = bb > 0.0 ? std::sqrt(rr / bb) : 0.0;
    {
        StageScope t(c, PIC_STAGE_PCG_FIELD, 2);
        pic::launch_fem_gradient(g, pcg_nbr(c, c->pcg_x), c->E4, halo_dst(c), c->partials, c->energies + 2 * slot,
                                 c->stream);
        PIC_LAUNCHED(c, "fem_gradient");
        c->pcg_launches += 2;
    }
    if (g.P > 1) {
        StageScope t(c, PIC_STAGE_EXCHANGE, 0);
        PIC_NCCL(c, ncclAllReduce(c->energies + 2 * slot, c->energies + 2 * slot, 2, ncclDouble, ncclSum,
                                  c->comm, c->stream));
    }
    c->last_slot = slot;
    if (!converged) {
        snprintf(c->err, sizeof(c->err), "FEM CG did not converge in %d iterations (relative residual %.3e)",
                 c->p.pcg_maxit, c->pcg_last_relres);
        return PIC_ENONCONV;
    }
    return PIC_OK;
}

// The field solve of the configured solver; rho = dscale * (the raw charge planes).
pic_status solve_field(pic_ctx* c, double dscale, int slot) {
    if (c->p.solver == PIC_SOLVER_PCG) return solve_pcg(c, dscale, slot);
    if (c->p.solver == PIC_SOLVER_FEM) return solve_fem(c, dscale, slot);
    return solve(c, dscale / ((double)c->g.n * c->g.n * c->g.n), slot);   // 1/N^3 of the whole box
}

// push=1: the step's push of the sorted state (with migration at P > 1);
// push=0: the state as is, any order.  The particles of buffer cur end sorted by
// cell key in cur^1 and their charge is deposited; cur flips.
pic_status push_sort_deposit(pic_ctx* c, int push) {
    const Geom& g = c->g;
    const bool peer_mig = push && g.P > 1 && c->mig_p2p;
    {
        StageScope t(c, PIC_STAGE_CLEAR, 0);
        PIC_CUDA(c, cudaMemsetAsync(c->count, 0, sizeof(uint32_t) * (size_t)c->ncell, c->stream));
        PIC_CUDA(c, cudaMemsetAsync(c->rho, 0, sizeof(double) * (size_t)g.nyr * g.rp * (g.nzl + 1), c->stream));
        if (g.P > 1) PIC_CUDA(c, cudaMemsetAsync(c->send_count, 0, sizeof(uint32_t) * g.P, c->stream));
        if (g.P > 1 && c->mig_p2p && !push) pic::launch_set_u64(c->dcnt + pic::DC_N, (unsigned long long)c->np, c->stream);
    }
    if (g.P > 1 && c->p2p && !push) {   // peers add ghost charge only after everyone cleared
        StageScope t(c, PIC_STAGE_EXCHANGE, 0);    // (in a step, the barrier after the push orders it)
        PIC_TRY(barrier(c));
    }
    PState cur = state(c, c->cur), nxt = state(c, c->cur ^ 1);
    pic::PeerRecv peers{};
    if (peer_mig) {
        for (int r = 0; r < g.P; ++r) {
            peers.peer_recv[r] = on_rank(c, r, c->recv);
            peers.peer_arr[r] = on_rank(c, r, c->dcnt + pic::DC_ARR);
        }
        peers.recv_cap = c->recv_cap;
    }
    {
        StageScope t(c, PIC_STAGE_PUSH_KEY, 1);
        if (push)
            pic::launch_push_key(g, cur, c->offs, c->E4, c->key, c->rank, c->count, c->send, c->send_count,
                                 c->segs, peer_mig ? &peers : nullptr, c->bprev, c->err_flag, c->stream);
        else
            pic::launch_key_import(g, cur, c->np, c->key, c->rank, c->count, c->err_flag, c->stream);
    }
    PIC_LAUNCHED(c, "push_key");
    if (peer_mig && pic::leavers_batched()) {
        StageScope t(c, PIC_STAGE_EXCHANGE, 2);
        pic::launch_leaver_copy(g, c->send, c->segs, c->send_count, c->recv_count, peers, c->err_flag, c->stream);
        PIC_LAUNCHED(c, "leaver_copy");
    }
    const int64_t n_old = c->np;
    int64_t narr = 0, nleave = 0, n_bound = n_old;
    const unsigned long long* dc = nullptr;
    if (peer_mig) {
        StageScope t(c, PIC_STAGE_EXCHANGE, 0);
        PIC_TRY(barrier(c));
        dc = c->dcnt;
        pic::launch_key_arrivals(g, c->recv, c->recv_cap, 0, c->key, c->rank, c->count, c->err_flag, dc, c->stream);
        PIC_LAUNCHED(c, "key_arrivals");
        n_bound = c->np_cap + c->recv_cap;
    } else if (push && g.P > 1) {
        StageScope t(c, PIC_STAGE_EXCHANGE, 0);
        PIC_NCCL(c, ncclAlltoAll(c->send_count, c->recv_count, 1, ncclUint32, c->comm, c->stream));
        uint32_t sc[8], rc[8];
        PIC_CUDA(c, cudaMemcpyAsync(sc, c->send_count, sizeof(uint32_t) * g.P, cudaMemcpyDeviceToHost, c->stream));
        PIC_CUDA(c, cudaMemcpyAsync(rc, c->recv_count, sizeof(uint32_t) * g.P, cudaMemcpyDeviceToHost, c->stream));
        PIC_CUDA(c, cudaStreamSynchronize(c->stream));
        int over = 0;
        for (int r = 0; r < g.P; ++r) {
            if (sc[r] > (uint32_t)c->segs.cap[r]) over = 1;
            nleave += sc[r];
            narr += rc[r];
        }
        if (narr > c->recv_cap) over = 1;
        int any = 0;
        PIC_TRY(agree_any(c, over, &any));       // every rank returns, none is left in the send/recv
        if (any)
            return fail(c, PIC_EOVERFLOW, over ? "migration send segment or receive buffer overflow"
                                               : "migration overflow on another rank");
        PIC_NCCL(c, ncclGroupStart());
        int64_t roff = 0;
        for (int r = 0; r < g.P; ++r) {
            if (r == g.rank) continue;
            if (sc[r])
                PIC_NCCL(c, ncclSend(c->send + (size_t)4 * c->segs.off[r], 8 * (size_t)sc[r], ncclDouble, r,
                                     c->comm, c->stream));
            if (rc[r])
                PIC_NCCL(c, ncclRecv(c->recv + 4 * roff, 8 * (size_t)rc[r], ncclDouble, r, c->comm, c->stream));
            roff += rc[r];
        }
        PIC_NCCL(c, ncclGroupEnd());
        pic::launch_key_arrivals(g, c->recv, narr, n_old, c->key, c->rank, c->count, c->err_flag, nullptr, c->stream);
        PIC_LAUNCHED(c, "key_arrivals");
        c->migrated += nleave;
        n_bound = n_old + narr;
    }
    const int64_t n_new = n_old - nleave + narr;
    if (!peer_mig && push && g.P > 1) {
        int any = 0;
        PIC_TRY(agree_any(c, n_new > c->np_cap, &any));
        if (any) return fail(c, PIC_EOVERFLOW, "a slab holds more particles than its capacity");
    } else if (!peer_mig && n_new > c->np_cap) {
        return fail(c, PIC_EOVERFLOW, "slab holds more particles than its capacity");
    }
    { StageScope t(c, PIC_STAGE_SCAN, 3); pic::launch_scan(c->count, c->offs, c->ncell, c->scan_scratch, c->stream, true); }
    PIC_LAUNCHED(c, "scan");
    { StageScope t(c, PIC_STAGE_PLACE, 1); pic::launch_place(c->key, c->rank, n_bound, c->offs, c->count, c->perm, dc, c->np_cap, c->err_flag, c->stream,
                                                                      &g, push ? c->bprev : nullptr); }
    PIC_LAUNCHED(c, "place");
    {
        StageScope t(c, PIC_STAGE_REORDER_DEPOSIT, 1);
        pic::launch_reorder_deposit(g, c->offs, c->perm, cur, c->recv, n_old, dc, nxt, push, c->rho, ghost_dst(c),
                                    push ? c->bprev : nullptr, c->err_flag, c->stream);
    }
    PIC_LAUNCHED(c, "reorder_deposit");
    if (peer_mig) {
        pic::launch_counts_update(g, c->dcnt, c->send_count, c->np_cap, c->err_flag, c->stream);
        PIC_LAUNCHED(c, "counts_update");
        c->np_stale = true;
    }
    if (g.P > 1) {
        StageScope t(c, PIC_STAGE_EXCHANGE, 0);
        if (c->ghost_p2p) PIC_TRY(barrier(c));      // ghost charge in place before the next solve
        else PIC_TRY(fold_rho_ghost(c));
    }
    c->cur ^= 1;
    if (!peer_mig) c->np = n_new;
    return PIC_OK;
}

pic_status sync_check(pic_ctx* c) {
    PIC_CUDA(c, cudaStreamSynchronize(c->stream));
    if (c->np_stale) {
        unsigned long long d[4];
        PIC_CUDA(c, cudaMemcpy(d, c->dcnt, sizeof(d), cudaMemcpyDeviceToHost));
        c->np = (int64_t)d[pic::DC_N];
        c->migrated = (int64_t)d[pic::DC_MIGRATED];
        c->np_stale = false;
    }
    int flag[3] = {0, 0, 0};
    PIC_CUDA(c, cudaMemcpy(flag, c->err_flag, sizeof(flag), cudaMemcpyDeviceToHost));
    if (flag[1]) {
        PIC_CUDA(c, cudaMemset(c->err_flag + 1, 0, sizeof(int)));
        return fail(c, PIC_EINVAL, "imported position outside [0, L) or outside this rank's slab");
    }
    if (flag[0] || flag[2]) {
        char what[256];
        snprintf(what, sizeof(what),
                 "capacity exceeded: > %d particles in one cell, or a slab / migration segment full (D#23, D#25)",
                 pic::reorder_cell_capacity(c->g.P));
        return fail(c, PIC_EOVERFLOW, what);
    }
    if (c->g.P > 1 && c->comm) {
        ncclResult_t ar = ncclSuccess;
        if (ncclCommGetAsyncError(c->comm, &ar) == ncclSuccess && ar != ncclSuccess) {
            snprintf(c->err, sizeof(c->err), "NCCL async error: %s", ncclGetErrorString(ar));
            c->poisoned = true;
            return PIC_ENCCL;
        }
    }
    if (c->timing) collect_timings(c);
    return PIC_OK;
}

// Domain grid [nzl][nyl][n] host <-> pitched device planes [nzl][nyr][rp] (pencils skip the
// ghost row of every plane).
pic_status copy_grid_to_device(pic_ctx* c, double* dst, const double* host) {
    const Geom& g = c->g;
    for (int z = 0; z < (g.Py > 1 ? g.nzl : 1); ++z)
        PIC_CUDA(c, cudaMemcpy2DAsync(dst + (size_t)z * g.nyr * g.rp, sizeof(double) * g.rp,
                                      host + (size_t)z * g.nyl * g.n, sizeof(double) * g.n, sizeof(double) * g.n,
                                      (size_t)g.nyl * (g.Py > 1 ? 1 : g.nzl), cudaMemcpyHostToDevice, c->stream));
    return PIC_OK;
}

pic_status copy_grid_to_host(pic_ctx* c, double* host, const double* src) {
    const Geom& g = c->g;
    for (int z = 0; z < (g.Py > 1 ? g.nzl : 1); ++z)
        PIC_CUDA(c, cudaMemcpy2DAsync(host + (size_t)z * g.nyl * g.n, sizeof(double) * g.n,
                                      src + (size_t)z * g.nyr * g.rp, sizeof(double) * g.rp, sizeof(double) * g.n,
                                      (size_t)g.nyl * (g.Py > 1 ? 1 : g.nzl), cudaMemcpyDeviceToHost, c->stream));
    return PIC_OK;
}

// Map every rank's workspace into this process (CUDA IPC; NVLink peer access) so the
// transposes, halo/ghost planes and migration become peer stores of the producing
// kernels.  Every rank must succeed, else all keep the NCCL transport; PIC_P2P=0 in
// the environment forces the NCCL transport.
pic_status setup_p2p(pic_ctx* c) {
    const Geom& g = c->g;
    c->peer_ws[g.rank] = c->ws;
    struct Rec {
        cudaIpcMemHandle_t h;
        long long off;
        long long lay[7];     // on_rank() needs the same carve on every rank
        int ok, pad;
    };
    Rec mine{};
    const long long lay[7] = {(long long)(reinterpret_cast<char*>(c->rho) - c->ws),
                              (long long)(reinterpret_cast<char*>(c->part[1][0]) - c->ws),
                              (long long)(reinterpret_cast<char*>(c->specA) - c->ws),
                              (long long)(reinterpret_cast<char*>(c->E4) - c->ws),
                              (long long)(reinterpret_cast<char*>(c->specD) - c->ws),
                              (long long)(reinterpret_cast<char*>(c->recv) - c->ws),
                              (long long)c->recv_cap};
    for (int k = 0; k < 7; ++k) mine.lay[k] = lay[k];
    const char* env = getenv("PIC_P2P");
    int ok = !(env && env[0] == '0');
    if (ok) {
        // the workspace may sit inside a larger allocation of the caller's allocator
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        typedef int (*GetRange)(unsigned long long*, size_t*, unsigned long long);
        unsigned long long base = 0;
        size_t sz = 0;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn ||
            reinterpret_cast<GetRange>(fn)(&base, &sz, (unsigned long long)c->ws) != 0 ||
            cudaIpcGetMemHandle(&mine.h, reinterpret_cast<void*>(base)) != cudaSuccess) {
            ok = 0;
        } else {
            mine.off = (long long)(c->ws - reinterpret_cast<char*>(base));
        }
        cudaGetLastError();
    }
    mine.ok = ok;
    char* dsend = reinterpret_cast<char*>(c->specC);    // free at init
    char* drecv = dsend + 256;
    std::vector<Rec> all(g.P);
    PIC_CUDA(c, cudaMemcpyAsync(dsend, &mine, sizeof(Rec), cudaMemcpyHostToDevice, c->stream));
    PIC_NCCL(c, ncclAllGather(dsend, drecv, sizeof(Rec), ncclUint8, c->comm, c->stream));
    PIC_CUDA(c, cudaMemcpyAsync(all.data(), drecv, sizeof(Rec) * g.P, cudaMemcpyDeviceToHost, c->stream));
    PIC_CUDA(c, cudaStreamSynchronize(c->stream));
    for (int r = 0; r < g.P; ++r) {
        ok = ok && all[r].ok;
        for (int k = 0; k < 7; ++k) ok = ok && all[r].lay[k] == lay[k];
    }
    for (int r = 0; r < g.P && ok; ++r) {
        if (r == g.rank) continue;
        void* ptr = nullptr;
        if (cudaIpcOpenMemHandle(&ptr, all[r].h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
            cudaGetLastError();
            ok = 0;
            break;
        }
        c->ipc_open[r] = ptr;
        c->peer_ws[r] = reinterpret_cast<char*>(ptr) + all[r].off;
    }
    int* flag = reinterpret_cast<int*>(dsend);
    PIC_CUDA(c, cudaMemcpyAsync(flag, &ok, sizeof(int), cudaMemcpyHostToDevice, c->stream));
    PIC_NCCL(c, ncclAllReduce(flag, flag, 1, ncclInt, ncclMin, c->comm, c->stream));
    int agreed = 0;
    PIC_CUDA(c, cudaMemcpyAsync(&agreed, flag, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    PIC_CUDA(c, cudaStreamSynchronize(c->stream));
    if (!agreed) {
        for (int r = 0; r < g.P; ++r)
            if (c->ipc_open[r]) { cudaIpcCloseMemHandle(c->ipc_open[r]); c->ipc_open[r] = nullptr; }
    }
    // pencils map the workspaces too, but only the FFT transposes and the y-group
    // redistributions use them (migration, halos and ghost folds stay NCCL)
    c->ipc = agreed != 0;
    c->p2p = c->ipc && !c->pencil;
    // migration through the peers' receive buffers: z-slabs with the peer transport; pencils
    // with PIC_PENCIL_MIG=1 (r02 at 512^3 on 2 x 2: exchange 1.35 -> 1.21 ms but the step
    // 20.6 -> 21.0 ms, the solve's pulls slower by 0.5 ms; off by default)
    const char* menv = getenv("PIC_PENCIL_MIG");
    c->mig_p2p = c->p2p || (c->ipc && c->pencil && menv && menv[0] == '1');
    c->xpose_p2p = c->p2p && env && env[0] == '2';
    if (c->ipc) {
        double2* tab[32] = {};
        for (int r = 0; r < g.P; ++r) {
            tab[r] = on_rank(c, r, c->specB);
            tab[8 + r] = on_rank(c, r, c->specD);
            tab[16 + r] = on_rank(c, r, c->specA);
            tab[24 + r] = on_rank(c, r, c->specC);
        }
        PIC_CUDA(c, cudaMemcpy(c->peer_tab, tab, sizeof(tab), cudaMemcpyHostToDevice));
    }
    // FFT transposes on the peer transport: copy-engine pulls by default (r02 at 512^3 on 4 GPUs:
    // 0.98 ms per step against 1.29 for ncclAlltoAll and 1.97 for the pull kernel);
    // PIC_XPOSE_PULL=0 keeps ncclAlltoAll, 1 the pull kernel
    const char* xenv = getenv("PIC_XPOSE_PULL");
    const char xm = xenv && xenv[0] ? xenv[0] : '2';
    c->xpose_pull = c->ipc && !c->xpose_p2p && (xm == '1' || xm == '2');
    c->xpose_ce = c->xpose_pull && xm == '2';
    // split transposes (r02, 512^3 on 4 GPUs): pencils 2 x 2 20.60 -> 20.45 ms, slabs 19.37 ->
    // 19.33 / 19.79 ms (no gain, more spread): on for pencils, PIC_XPOSE_SPLIT=0/1 overrides
    const char* senv = getenv("PIC_XPOSE_SPLIT");
    c->xpose_split = c->xpose_ce && (senv && senv[0] ? senv[0] == '1' : c->pencil);
    const char* penv = getenv("PIC_PENCIL_PULL");          // 0: the NCCL y-group all-to-alls
    c->pen_ce = c->ipc && c->pencil && !(penv && penv[0] == '0');
    if (c->xpose_ce || c->pen_ce) {
        for (int r = 0; r < g.P; ++r) {
            PIC_CUDA(c, cudaStreamCreateWithFlags(&c->side[r], cudaStreamNonBlocking));
            PIC_CUDA(c, cudaEventCreateWithFlags(&c->side_ev[r], cudaEventDisableTiming));
        }
        PIC_CUDA(c, cudaEventCreateWithFlags(&c->side_ev[8], cudaEventDisableTiming));
    }
    const char* genv = getenv("PIC_P2P_GHOST");
    c->ghost_p2p = c->p2p && genv && genv[0] == '2';
    return PIC_OK;
}


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
    p->solver = PIC_SOLVER_FFT;
    p->pcg_inner = 4;
    p->pcg_outer = 2;
    p->pcg_maxit = 10000;         // plain CG (FEM) needs ~N iterations
    p->pcg_tol = 1e-4;
    p->pcg_omega = M_PI / 2;      // P:260 "damping factor of pi/2"
    return PIC_OK;
}

pic_status pic_nccl_unique_id(uint8_t* id) {
    if (!id) return PIC_EINVAL;
    ncclUniqueId u;
    if (ncclGetUniqueId(&u) != ncclSuccess) return PIC_ENCCL;
    static_assert(sizeof(u) <= 128, "ncclUniqueId larger than 128 bytes");
    std::memset(id, 0, 128);
    std::memcpy(id, &u, sizeof(u));
    return PIC_OK;
}

pic_status pic_workspace_bytes(const pic_params* p, int32_t rank, int32_t nranks, size_t* bytes) {
    char msg[256];
    pic_status st = validate(p, rank, nranks, msg, sizeof(msg));
    if (st != PIC_OK) { snprintf(g_init_error, sizeof(g_init_error), "%s", msg); return st; }
    if (!bytes) return PIC_EINVAL;
    const Geom g = make_geom(p, rank, nranks);
    const Sizes z = sizes(p, g);
    if ((st = validate_sizes(z, msg, sizeof(msg))) != PIC_OK) {
        snprintf(g_init_error, sizeof(g_init_error), "%s", msg);
        return st;
    }
    *bytes = carve(nullptr, g, z, nullptr);
    return PIC_OK;
}

pic_status pic_slab(const pic_params* p, int32_t rank, int32_t nranks, int32_t* z0, int32_t* nz,
                    int64_t* capacity) {
    char msg[256];
    pic_status st = validate(p, rank, nranks, msg, sizeof(msg));
    if (st != PIC_OK) { snprintf(g_init_error, sizeof(g_init_error), "%s", msg); return st; }
    const Geom g = make_geom(p, rank, nranks);
    if (z0) *z0 = g.z0;
    if (nz) *nz = g.nzl;
    if (capacity) *capacity = sizes(p, g).np_cap;
    return PIC_OK;
}

pic_status pic_domain(const pic_params* p, int32_t rank, int32_t nranks, int32_t* y0, int32_t* ny, int32_t* z0,
                      int32_t* nz, int64_t* capacity) {
    char msg[256];
    pic_status st = validate(p, rank, nranks, msg, sizeof(msg));
    if (st != PIC_OK) { snprintf(g_init_error, sizeof(g_init_error), "%s", msg); return st; }
    const Geom g = make_geom(p, rank, nranks);
    if (y0) *y0 = g.y0;
    if (ny) *ny = g.nyl;
    if (z0) *z0 = g.z0;
    if (nz) *nz = g.nzl;
    if (capacity) *capacity = sizes(p, g).np_cap;
    return PIC_OK;
}

pic_status pic_init(const pic_params* p, int32_t rank, int32_t nranks, const uint8_t* nccl_id,
                    void* workspace, size_t workspace_bytes, void* cuda_stream, pic_ctx** out) {
    if (!out) return PIC_EINVAL;
    *out = nullptr;
    char msg[256];
    pic_status st = validate(p, rank, nranks, msg, sizeof(msg));
    if (st != PIC_OK) { snprintf(g_init_error, sizeof(g_init_error), "%s", msg); return st; }
    if (nranks > 1 && !nccl_id) {
        snprintf(g_init_error, sizeof(g_init_error), "nccl_id required for nranks > 1");
        return PIC_EINVAL;
    }
    const Geom g = make_geom(p, rank, nranks);
    const Sizes z = sizes(p, g);
    if ((st = validate_sizes(z, msg, sizeof(msg))) != PIC_OK) {
        snprintf(g_init_error, sizeof(g_init_error), "%s", msg);
        return st;
    }
    const size_t need = carve(nullptr, g, z, nullptr);
    if (!workspace || workspace_bytes < need) {
        snprintf(g_init_error, sizeof(g_init_error), "workspace %zu B < %zu B needed", workspace_bytes, need);
        return PIC_ENOMEM;
    }
    pic_ctx* c = new (std::nothrow) pic_ctx();
    if (!c) return PIC_ENOMEM;
    c->p = *p;
    c->g = g;
    c->g.cap = z.np_cap;
    c->gs = slab_geom(c->g);
    c->pencil = g.Py > 1;
    c->ws = reinterpret_cast<char*>(workspace);
    c->np_glob = (int64_t)p->ppc * p->n * p->n * p->n;
    c->ncell = (int64_t)g.n * g.nyl * g.nzl;
    c->q = -((g.L * g.L) * g.L) / (double)c->np_glob;
    c->deposit_scale = c->q * ((g.inv_h * g.inv_h) * g.inv_h);
    c->stream = reinterpret_cast<cudaStream_t>(cuda_stream);
    carve(c, c->g, z, reinterpret_cast<char*>(workspace));

    // the dynamic shared-memory opt-in is a per-device attribute: set it once per device
    static unsigned smem_set = 0;      // bit d: device d done
    {
        int dev = 0;
        cudaError_t e0 = cudaGetDevice(&dev);
        if (e0 == cudaSuccess && dev < 32 && !(smem_set & (1u << dev))) {
            e0 = pic::fft_set_smem_limits();
            if (e0 == cudaSuccess) e0 = pic::particles_set_smem_limits();
            if (e0 == cudaSuccess) smem_set |= 1u << dev;
        }
        if (e0 != cudaSuccess) {
            snprintf(g_init_error, sizeof(g_init_error), "shared-memory opt-in: %s", cudaGetErrorString(e0));
            delete c;
            return PIC_ECUDA;
        }
    }

    auto bail = [&](pic_status s) {
        snprintf(g_init_error, sizeof(g_init_error), "%s", c->err);
        for (int r = 0; r < 8; ++r)
            if (c->ipc_open[r]) cudaIpcCloseMemHandle(c->ipc_open[r]);
        if (c->ycomm) ncclCommDestroy(c->ycomm);
        if (c->comm) ncclCommDestroy(c->comm);
        delete c;
        return s;
    };
    if (nranks > 1) {
        ncclUniqueId u;
        std::memcpy(&u, nccl_id, sizeof(u));
        ncclResult_t r = ncclCommInitRank(&c->comm, nranks, u, rank);
        if (r != ncclSuccess) {
            snprintf(c->err, sizeof(c->err), "ncclCommInitRank: %s", ncclGetErrorString(r));
            return bail(PIC_ENCCL);
        }
        if (c->pencil) {
            // the y-group (ranks sharing pz) for the pencil <-> slab redistributions (NCCL
            // fallback); pencils keep the NCCL transport for migration, halos and ghost folds
            r = ncclCommSplit(c->comm, rank / g.Py, rank % g.Py, &c->ycomm, nullptr);
            if (r != ncclSuccess) {
                snprintf(c->err, sizeof(c->err), "ncclCommSplit: %s", ncclGetErrorString(r));
                return bail(PIC_ENCCL);
            }
        }
        if ((st = setup_p2p(c)) != PIC_OK) return bail(st);
        if (p->solver != PIC_SOLVER_FFT && !c->p2p) {
            snprintf(c->err, sizeof(c->err), "the PCG / FEM solvers at P > 1 need the peer-memory transport");
            return bail(PIC_EUNSUPPORTED);
        }
    }
    if (c->pcg_x) {   // warm start of the first solve: phi = 0
        cudaError_t e0 = cudaMemsetAsync(c->pcg_x, 0, sizeof(double) * (size_t)c->ncell, c->stream);
        if (e0 != cudaSuccess) return bail(fail(c, PIC_ECUDA, "pcg init", e0));
    }
    // twiddles W_n^m = exp(-2 pi i m / n), m < n
    std::vector<double2> tw(g.n);
    for (int m = 0; m < g.n; ++m) {
        const double ang = 2.0 * M_PI * (double)m / (double)g.n;
        tw[m] = make_double2(std::cos(ang), -std::sin(ang));
    }
    cudaError_t e = cudaMemcpyAsync(c->tw, tw.data(), sizeof(double2) * tw.size(), cudaMemcpyHostToDevice, c->stream);
    if (e == cudaSuccess) e = cudaMemsetAsync(c->err_flag, 0, sizeof(int) * 4, c->stream);
    if (e == cudaSuccess) e = cudaMemsetAsync(c->dcnt, 0, sizeof(unsigned long long) * 4, c->stream);
    if (e != cudaSuccess) return bail(fail(c, PIC_ECUDA, "init copies", e));

    if (g.P == 1) {
        c->np = c->np_glob;
        pic::launch_sample(g, state(c, 0), c->np, p->k, p->alpha, p->seed, c->stream);
    } else {
        // every rank samples the z coordinate of every global index j and keeps its own,
        // in ascending j (the oracle's initial order restricted to the slab)
        const int64_t nblk = pic::sample_blocks(c->np_glob);
        pic::launch_sample_count(g, c->np_glob, p->k, p->alpha, p->seed, c->key, c->stream);
        pic::launch_scan(c->key, c->perm, nblk, c->scan_scratch, c->stream);
        uint32_t total = 0;
        e = cudaMemcpyAsync(&total, c->perm + nblk, sizeof(uint32_t), cudaMemcpyDeviceToHost, c->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
        if (e != cudaSuccess) return bail(fail(c, PIC_ECUDA, "sample count", e));
        int any = 0;
        if ((st = agree_any(c, (int64_t)total > c->np_cap, &any)) != PIC_OK) return bail(st);
        if (any) return bail(fail(c, PIC_EOVERFLOW, "slab capacity exceeded at init (on this or another rank)"));
        c->np = total;
        pic::launch_sample_write(g, state(c, 0), c->np_glob, p->k, p->alpha, p->seed, c->perm, c->stream);
    }
    e = cudaGetLastError();
    if (e != cudaSuccess) return bail(fail(c, PIC_ECUDA, "sample", e));
    c->cur = 0;
    if ((st = push_sort_deposit(c, 0)) != PIC_OK) return bail(st);
    if (p->half_kick) {
        if ((st = solve_field(c, c->deposit_scale, 0)) != PIC_OK) return bail(st);
        pic::launch_half_kick(g, state(c, c->cur), c->np, c->E4, c->stream);
        e = cudaGetLastError();
        if (e != cudaSuccess) return bail(fail(c, PIC_ECUDA, "half_kick", e));
        c->last_slot = -1;
        // the solve reused the charge buffer: deposit again (the re-sort is the identity)
        if ((st = push_sort_deposit(c, 0)) != PIC_OK) return bail(st);
    }
    if ((st = sync_check(c)) != PIC_OK) return bail(st);
    c->migrated = 0;
    if (c->mig_p2p) {
        pic::launch_set_u64(c->dcnt + pic::DC_MIGRATED, 0ull, c->stream);
        if ((st = sync_check(c)) != PIC_OK) return bail(st);
    }
    *out = c;
    return PIC_OK;
}

pic_status pic_step(pic_ctx* c, int32_t nsteps, double* ex_energy) {
    PIC_CHECK_CTX(c);
    if (nsteps < 0) return PIC_EINVAL;
    int32_t done = 0;
    while (done < nsteps) {
        const int chunk = std::min(nsteps - done, kMaxEnergySteps);
        for (int s = 0; s < chunk; ++s) {
            PIC_TRY(solve_field(c, c->deposit_scale, s));
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
    for (int r = 0; r < 8; ++r) {
        if (c->side[r]) cudaStreamDestroy(c->side[r]);
        if (c->side_ev[r]) cudaEventDestroy(c->side_ev[r]);
    }
    if (c->side_ev[8]) cudaEventDestroy(c->side_ev[8]);
    for (int r = 0; r < 8; ++r)
        if (c->ipc_open[r]) cudaIpcCloseMemHandle(c->ipc_open[r]);
    if (c->ycomm) ncclCommDestroy(c->ycomm);
    if (c->comm) ncclCommDestroy(c->comm);
    delete c;
}

const char* pic_last_error(const pic_ctx* c) { return c ? c->err : g_init_error; }

pic_status pic_num_particles(pic_ctx* c, int64_t* np) {
    if (!c || !np) return PIC_EINVAL;
    *np = c->np;
    return PIC_OK;
}

pic_status pic_migrated(pic_ctx* c, int64_t* migrated) {
    if (!c || !migrated) return PIC_EINVAL;
    *migrated = c->migrated;
    return PIC_OK;
}

pic_status pic_peer_transport(pic_ctx* c, int32_t* peer) {
    if (!c || !peer) return PIC_EINVAL;
    *peer = c->p2p ? 1 : 0;
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

pic_status pic_gather_particles(pic_ctx* c, double* xyzuvw, int64_t np_total, int64_t* np_out) {
    PIC_CHECK_CTX(c);
    const Geom& g = c->g;
    if (g.P == 1) {
        if (np_out) *np_out = c->np;
        if (!xyzuvw) return PIC_OK;
        return pic_get_particles(c, xyzuvw, np_total);
    }
    PIC_TRY(sync_check(c));               // np up to date (peer transport: device counts)
    // every rank's count (int64) -> all ranks
    int64_t* dcounts = reinterpret_cast<int64_t*>(c->specC);     // scratch outside a solve
    int64_t mine = c->np;
    std::vector<int64_t> counts(g.P);
    PIC_CUDA(c, cudaMemcpyAsync(dcounts + 8, &mine, sizeof(int64_t), cudaMemcpyHostToDevice, c->stream));
    PIC_NCCL(c, ncclAllGather(dcounts + 8, dcounts, 1, ncclInt64, c->comm, c->stream));
    PIC_CUDA(c, cudaMemcpyAsync(counts.data(), dcounts, sizeof(int64_t) * g.P, cudaMemcpyDeviceToHost, c->stream));
    PIC_CUDA(c, cudaStreamSynchronize(c->stream));
    int64_t total = 0;
    for (int r = 0; r < g.P; ++r) total += counts[r];
    if (np_out) *np_out = total;
    int want = 0;                          // rank 0 decides whether to gather, every rank follows
    if (g.rank == 0) want = xyzuvw ? (np_total == total ? 1 : 2) : 0;
    int* dflag = c->bar + 3;
    PIC_CUDA(c, cudaMemcpyAsync(dflag, &want, sizeof(int), cudaMemcpyHostToDevice, c->stream));
    PIC_NCCL(c, ncclBroadcast(dflag, dflag, 1, ncclInt, 0, c->comm, c->stream));
    PIC_CUDA(c, cudaMemcpyAsync(&want, dflag, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    PIC_CUDA(c, cudaStreamSynchronize(c->stream));
    if (want == 0) return PIC_OK;
    if (want == 2) {
        snprintf(c->err, sizeof(c->err), "pic_gather_particles: np_total %lld != %lld particles on all ranks",
                 (long long)np_total, (long long)total);
        return PIC_EINVAL;
    }
    // this rank's canonical SoA [6][np_r] in its idle buffer; rank 0 copies its own, then
    // receives rank r's into the same buffer (every rank's np_r <= the common capacity)
    double* soa = reinterpret_cast<double*>(c->part[c->cur ^ 1][0]);
    pic::launch_pairs_to_soa(state(c, c->cur), c->np, soa, c->stream);
    PIC_LAUNCHED(c, "pairs_to_soa");
    int64_t off = 0;
    for (int r = 0; r < g.P; ++r) {
        const int64_t nr = counts[r];
        if (r > 0 && nr > 0) {
            PIC_NCCL(c, ncclGroupStart());
            if (g.rank == r) PIC_NCCL(c, ncclSend(soa, (size_t)(6 * nr), ncclDouble, 0, c->comm, c->stream));
            if (g.rank == 0) PIC_NCCL(c, ncclRecv(soa, (size_t)(6 * nr), ncclDouble, r, c->comm, c->stream));
            PIC_NCCL(c, ncclGroupEnd());
        }
        if (g.rank == 0 && nr > 0) {
            PIC_CUDA(c, cudaMemcpy2DAsync(xyzuvw + off, sizeof(double) * (size_t)total, soa, sizeof(double) * (size_t)nr,
                                          sizeof(double) * (size_t)nr, 6, cudaMemcpyDeviceToHost, c->stream));
            PIC_CUDA(c, cudaStreamSynchronize(c->stream));   // the buffer is reused for the next rank
        }
        off += nr;
    }
    PIC_TRY(sync_check(c));
    if (g.rank != 0 || total == 0) return PIC_OK;
    // global canonical order: stable counting sort by the global Morton cell key (D#5, D#14)
    const int64_t ncell = (int64_t)g.n * g.n * g.n;
    auto cell = [&](double x) {
        int i = (int)std::floor(x * g.inv_h);
        return i > g.n - 1 ? g.n - 1 : (i < 0 ? 0 : i);
    };
    auto morton = [&](int ix, int iy, int iz) {
        uint32_t k = 0;
        for (int b = 0; (1 << b) < g.n; ++b)
            k |= ((uint32_t)((ix >> b) & 1) << (3 * b)) | ((uint32_t)((iy >> b) & 1) << (3 * b + 1)) |
                 ((uint32_t)((iz >> b) & 1) << (3 * b + 2));
        return k;
    };
    std::vector<uint32_t> key((size_t)total);
    for (int64_t j = 0; j < total; ++j)
        key[j] = morton(cell(xyzuvw[j]), cell(xyzuvw[total + j]), cell(xyzuvw[2 * total + j]));
    std::vector<int64_t> start((size_t)ncell + 1, 0);
    for (int64_t j = 0; j < total; ++j) start[key[j] + 1] += 1;
    for (int64_t k = 0; k < ncell; ++k) start[k + 1] += start[k];
    std::vector<int64_t> dst((size_t)total);
    for (int64_t j = 0; j < total; ++j) dst[j] = start[key[j]]++;
    std::vector<double> tmp((size_t)total);
    for (int a = 0; a < 6; ++a) {
        double* col = xyzuvw + (int64_t)a * total;
        for (int64_t j = 0; j < total; ++j) tmp[dst[j]] = col[j];
        std::memcpy(col, tmp.data(), sizeof(double) * (size_t)total);
    }
    return PIC_OK;
}

pic_status pic_owner_ranks(const pic_params* p, int32_t nranks, const double* xyz, int64_t np, int32_t* owner) {
    char msg[256];
    pic_status st = validate(p, 0, nranks, msg, sizeof(msg));
    if (st != PIC_OK) { snprintf(g_init_error, sizeof(g_init_error), "%s", msg); return st; }
    if (np < 0 || (np > 0 && (!xyz || !owner))) return PIC_EINVAL;
    const Geom g = make_geom(p, 0, nranks);
    const double* y = xyz + np;
    const double* z = xyz + 2 * np;
    for (int64_t j = 0; j < np; ++j) {
        if (!(z[j] >= 0.0 && z[j] < g.L) || !(y[j] >= 0.0 && y[j] < g.L)) {
            snprintf(g_init_error, sizeof(g_init_error), "pic_owner_ranks: y/z[%lld] outside [0, L)", (long long)j);
            return PIC_EINVAL;
        }
        int iz = (int)std::floor(z[j] * g.inv_h);      // D#5: floor(x inv_h), clamped to N - 1
        iz = iz > g.n - 1 ? g.n - 1 : iz;
        int iy = (int)std::floor(y[j] * g.inv_h);
        iy = iy > g.n - 1 ? g.n - 1 : iy;
        owner[j] = (iz / g.nzl) * g.Py + iy / g.nyl;   // rank = pz Py + py (slabs: Py = 1)
    }
    return PIC_OK;
}

pic_status pic_set_particles(pic_ctx* c, const double* xyzuvw, int64_t np) {
    PIC_CHECK_CTX(c);
    if (!xyzuvw || np < 0 || np > c->np_cap || (c->g.P == 1 && np != c->np_glob)) return PIC_EINVAL;
    double* soa = reinterpret_cast<double*>(c->part[c->cur ^ 1][0]);
    PIC_CUDA(c, cudaMemcpyAsync(soa, xyzuvw, sizeof(double) * 6 * (size_t)np, cudaMemcpyHostToDevice, c->stream));
    pic::launch_soa_to_pairs(soa, np, state(c, c->cur), c->stream);
    PIC_LAUNCHED(c, "soa_to_pairs");
    c->np = np;
    if (c->pcg_x)      // PCG: the imported state restarts from phi = 0 (like pic_init)
        PIC_CUDA(c, cudaMemsetAsync(c->pcg_x, 0, sizeof(double) * (size_t)c->ncell, c->stream));
    PIC_TRY(push_sort_deposit(c, 0));
    c->last_slot = -1;
    return sync_check(c);
}

pic_status pic_get_grid(pic_ctx* c, int32_t which, double* host) {
    PIC_CHECK_CTX(c);
    bind_spec(c);
    if (!host || which < 0 || which > 4 || (which == 4 && !c->pcg_x)) return PIC_EINVAL;
    if (which == 0) {
        PIC_TRY(copy_grid_to_host(c, host, c->rho));
    } else if (which == 4) {
        double* scratch = reinterpret_cast<double*>(c->specC);
        if (c->p.solver == PIC_SOLVER_PCG) {
            pic::launch_pcg_unsplit(c->g, c->pcg_x, scratch, c->stream);
            PIC_LAUNCHED(c, "pcg_unsplit");
        } else {
            scratch = c->pcg_x;     // FEM: natural layout already
        }
        PIC_CUDA(c, cudaMemcpyAsync(host, scratch, sizeof(double) * (size_t)c->ncell,
                                    cudaMemcpyDeviceToHost, c->stream));
    } else {
        double* scratch = reinterpret_cast<double*>(c->specC);
        pic::launch_e4_extract(c->g, c->E4, which - 1, scratch, c->stream);
        PIC_LAUNCHED(c, "e4_extract");
        PIC_CUDA(c, cudaMemcpyAsync(host, scratch, sizeof(double) * (size_t)c->ncell,
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
    if (c->pcg_x)      // PCG: solve from phi = 0 (the particles' warm start is reset too)
        PIC_CUDA(c, cudaMemsetAsync(c->pcg_x, 0, sizeof(double) * (size_t)c->ncell, c->stream));
    PIC_TRY(solve_field(c, 1.0, 0));
    double en[2];
    PIC_CUDA(c, cudaMemcpyAsync(en, c->energies, sizeof(en), cudaMemcpyDeviceToHost, c->stream));
    if (E_host) {
        bind_spec(c);
        double* scratch = reinterpret_cast<double*>(c->specC);
        for (int d = 0; d < 3; ++d) {
            pic::launch_e4_extract(c->g, c->E4, d, scratch, c->stream);
            PIC_LAUNCHED(c, "e4_extract");
            PIC_CUDA(c, cudaMemcpyAsync(E_host + (size_t)d * c->ncell, scratch, sizeof(double) * (size_t)c->ncell,
                                        cudaMemcpyDeviceToHost, c->stream));
        }
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
    bind_spec(c);
    if (!E_host) return PIC_EINVAL;
    double* sc = reinterpret_cast<double*>(c->specC);   // scratch: 3 compact slab components
    double* const comp[3] = {sc, sc + c->ncell, sc + 2 * c->ncell};
    for (int d = 0; d < 3; ++d)
        PIC_CUDA(c, cudaMemcpyAsync(comp[d], E_host + (size_t)d * c->ncell, sizeof(double) * (size_t)c->ncell,
                                    cudaMemcpyHostToDevice, c->stream));
    pic::launch_e4_pack(c->g, comp, c->E4, c->stream);
    PIC_LAUNCHED(c, "e4_pack");
    PIC_TRY(refresh_halo(c));
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
        pic::launch_gkeys(c->g, state(c, c->cur), c->np, c->key, c->stream);
        PIC_LAUNCHED(c, "gkeys");
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
    // solve 6, push_key 1, scan 3, place 1, reorder_deposit 1; P > 1: arrivals 1, and
    // the NCCL transport's ghost fold 1 or the peer transport's count update 1
    // pencils: + the ghost row fold and the field's pack / unpack around the y-group all-to-all
    *launches = 12 + (c->g.P > 1 ? 2 : 0) + (c->g.P > 1 && c->mig_p2p && pic::leavers_batched() ? 2 : 0) +
                (c->pencil ? (c->pen_ce ? 1 : 3) : 0) + (xpose_split(c) ? 2 : 0);
    if (c->p.solver != PIC_SOLVER_FFT) *launches += c->pcg_launches - 6;   // the latest CG solve's count
    return PIC_OK;
}

pic_status pic_diag_bandwidth(pic_ctx* c, int32_t mode, int32_t reps, double* ms, double* bytes) {
    PIC_CHECK_CTX(c);
    if (reps < 1 || mode < 0 || mode > 3) return PIC_EINVAL;
    PIC_TRY(sync_check(c));
    cudaEvent_t e0, e1;
    PIC_CUDA(c, cudaEventCreate(&e0));
    PIC_CUDA(c, cudaEventCreate(&e1));
    double b = 0.0;
    PIC_CUDA(c, cudaEventRecord(e0, c->stream));
    for (int r = 0; r < reps; ++r)
        b = pic::launch_diag(mode, state(c, c->cur), state(c, c->cur ^ 1), c->perm, c->key, c->np,
                             c->partials, c->stream);
    PIC_CUDA(c, cudaEventRecord(e1, c->stream));
    PIC_CUDA(c, cudaEventSynchronize(e1));
    float t = 0.f;
    PIC_CUDA(c, cudaEventElapsedTime(&t, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    PIC_LAUNCHED(c, "diag");
    if (ms) *ms = t / reps;
    if (bytes) *bytes = b;
    return PIC_OK;
}

pic_status pic_pcg_stats(pic_ctx* c, int32_t* last_iters, int64_t* total_iters, int64_t* solves,
                         double* last_relres) {
    if (!c) return PIC_EINVAL;
    if (c->p.solver == PIC_SOLVER_FFT) { snprintf(c->err, sizeof(c->err), "not a PCG / FEM context"); return PIC_EINVAL; }
    if (last_iters) *last_iters = c->pcg_last_iters;
    if (total_iters) *total_iters = c->pcg_total_iters;
    if (solves) *solves = c->pcg_solves;
    if (last_relres) *last_relres = c->pcg_last_relres;
    return PIC_OK;
}

}  // extern "C"
