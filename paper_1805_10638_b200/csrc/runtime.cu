// runtime.cu -- host runtime + C ABI of libaakm.so (include/aakm.h).
//
// One Algorithm 1 pass is enqueued as a fixed kernel
// sequence whose data-dependent branches (converge / reject) are device
// predicates (aa.cu), so the same sequence can be launched eagerly or
// captured once into a CUDA graph and replayed until the device sets `done`.
// Multi-rank: one ncclAllReduce(sum, int64) of the packed exact fixed-point
// [S_hi|S_lo|N|E_hi|E_lo|E|changed] vector per G-evaluation, issued in-stream
// (and captured in the graph).
#include <cuda_runtime.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <string>
#include <algorithm>
#include <chrono>
#include <mutex>
#include <thread>
#include <vector>

#include "../../include/aakm.h"
#include "aakm_dev.cuh"

using namespace aakm;

struct kmeans_handle {
    Dev d;          // Algorithm 1 state and buffers
    Dev da;         // API calls (assign/update): own DevState + centroid buffers
    kmeans_config cfg;
    cudaStream_t stream = nullptr;
    int rank = 0, nranks = 1;
    long long n_global = 0;
    ncclComm_t comm = nullptr;
    bool poisoned = false;
    std::string err;
    int path = KMEANS_PATH_SIMT;
    size_t scratch_bytes = 0;
    void* scratch = nullptr;
    cudaGraphExec_t pass_exec = nullptr;
    cudaStream_t cap_stream = nullptr;   // private non-blocking stream used only for graph capture
    void* tcm = nullptr;                 // TMA maps for d (tensor-core engine)
    void* tcm_api = nullptr;             // TMA maps for da
    long long launches = 0;
    long long kernels_per_pass = 0;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev;   // assignment timing (branch A)
    size_t ev_used = 0;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> uev;  // update timing (branch A)
    size_t uev_used = 0;
    DevState* st_host = nullptr;                             // pinned
    TraceRec* tr_host = nullptr;                             // pinned
    double* scal_host = nullptr;                             // pinned (E, changed)
    float x_gamax = 0.f;                                     // max |x_ik| over all ranks (K-Means++ scale)
    // streamed X (kmeans_aa_step_host): H2D row chunks on copy_stream, one event each
    cudaStream_t copy_stream = nullptr;
    std::vector<cudaEvent_t> feed_ev;
    cudaEvent_t feed_gate = nullptr, feed_all = nullptr;
    int feed_chunks = 0;                                     // > 0 while a streamed pass is enqueued
    long long feed_tiles = 0;                                // row tiles per chunk (even)
    cudaEvent_t run_ev[2] = {nullptr, nullptr};
    int* done_host = nullptr;                                // pinned
    unsigned int* xchk = nullptr;                            // device, 2 words: stats of a refreshed X
    unsigned int x_stat[2] = {0u, 0u};                       // this rank's create-time max |x|, max ||x||^2 (float bits)
    cudaEvent_t sync_ev = nullptr;                           // polled by sync_stream when a communicator exists
    cudaStream_t body_stream = nullptr;                      // capture of the conditional branch-B body
    long long kernels_b = 0;                                 // kernels inside it (launched only on rejections)
    std::vector<size_t> guards;                              // AAKM_WS_CANARY: canary offsets in the workspace
    char* ws_base = nullptr;
    void* fused = nullptr;                                   // f4 fused combine resources (comm.cu)
};

// NVTX ranges (SURVEY §5 tracing): one per API call and per Algorithm 1 step as it
// is enqueued -- the eager launches of aa_step / assign / update / seed_pp sit
// inside them (ncu --nvtx --nvtx-include "aakm:assign/" selects one step's
// kernels); under graph capture they mark the capture.  No-ops without a tool.
struct Nvtx {
    explicit Nvtx(const char* name) { nvtxRangePushA(name); }
    ~Nvtx() { nvtxRangePop(); }
    Nvtx(const Nvtx&) = delete;
    Nvtx& operator=(const Nvtx&) = delete;
};
// consecutive steps inside one scope: to() closes the open range and opens the next
struct NvtxStep {
    bool on = false;
    void to(const char* name) { if (on) nvtxRangePop(); nvtxRangePushA(name); on = true; }
    ~NvtxStep() { if (on) nvtxRangePop(); }
};

static thread_local std::string g_create_err;
static bool g_dbg = getenv("AAKM_DEBUG_SYNC") != nullptr;
static bool g_prof = getenv("AAKM_PROFILE") != nullptr;

// AAKM_PROFILE=1 (eager launches only): per-kernel CUDA-event durations,
// printed to stderr by kmeans_destroy.
struct ProfRec { const char* name; cudaEvent_t a, b; };
static std::vector<ProfRec> g_prof_recs;
static cudaEvent_t g_prof_last = nullptr;
static void prof_mark(const char* what, cudaStream_t s) {
    cudaStreamCaptureStatus cs;
    if (cudaStreamIsCapturing(s, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, s);
    if (g_prof_last) g_prof_recs.push_back({what, g_prof_last, e});
    g_prof_last = e;
}
static void prof_dump() {
    if (g_prof_recs.empty()) return;
    cudaDeviceSynchronize();
    std::vector<std::pair<std::string, std::pair<double, int>>> agg;
    for (auto& r : g_prof_recs) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, r.a, r.b);
        bool f = false;
        for (auto& a : agg) if (a.first == r.name) { a.second.first += ms; a.second.second++; f = true; }
        if (!f) agg.push_back({r.name, {ms, 1}});
    }
    fprintf(stderr, "[aakm prof] kernel            total_ms    calls   avg_ms\n");
    for (auto& a : agg)
        fprintf(stderr, "[aakm prof] %-16s %10.3f %8d %9.4f\n", a.first.c_str(), a.second.first, a.second.second,
                a.second.first / a.second.second);
    g_prof_recs.clear();
    g_prof_last = nullptr;
}

// AAKM_DEBUG_SYNC=1: synchronise after every launch and name the failing kernel.
static void dbg(const char* what, cudaStream_t s) {
    if (g_prof) prof_mark(what, s);
    if (!g_dbg) return;
    cudaError_t e = cudaStreamSynchronize(s);
    if (e == cudaSuccess) e = cudaGetLastError();
    fprintf(stderr, "[aakm dbg] %-16s %s\n", what, cudaGetErrorString(e));
}

#define FAIL(h, code, msg)                    \
    do {                                      \
        (h)->err = (msg);                     \
        if ((code) == KMEANS_ERR_CUDA || (code) == KMEANS_ERR_NCCL) (h)->poisoned = true; \
        return (code);                        \
    } while (0)

#define CK(h, call)                                                                        \
    do {                                                                                   \
        cudaError_t e_ = (call);                                                           \
        if (e_ != cudaSuccess) {                                                           \
            (h)->err = std::string(#call) + ": " + cudaGetErrorString(e_);                 \
            (h)->poisoned = true;                                                          \
            return KMEANS_ERR_CUDA;                                                        \
        }                                                                                  \
    } while (0)

#define NK(h, call)                                                                        \
    do {                                                                                   \
        ncclResult_t r_ = (call);                                                          \
        if (r_ != ncclSuccess) {                                                           \
            (h)->err = std::string(#call) + ": " + ncclGetErrorString(r_);                 \
            (h)->poisoned = true;                                                          \
            return KMEANS_ERR_NCCL;                                                        \
        }                                                                                  \
    } while (0)

// Wait for the stream.  With a communicator, poll instead of blocking: a peer
// that failed (ncclCommGetAsyncError) or a collective that does not complete
// within AAKM_COMM_TIMEOUT_S seconds (default 600) aborts the communicator and
// poisons the handle, so kmeans_run cannot hang forever on a dead rank.
static kmeans_status sync_stream(kmeans_handle* h, cudaStream_t s);
#define SYNC(h, s)                                                                         \
    do {                                                                                   \
        kmeans_status r_ = sync_stream((h), (s));                                          \
        if (r_ != KMEANS_OK) return r_;                                                    \
    } while (0)

#define LIVE(h)                                                                            \
    do {                                                                                   \
        if (!(h)) return KMEANS_ERR_INVALID;                                               \
        if ((h)->poisoned) { (h)->err = "handle poisoned by an earlier CUDA/NCCL error"; return KMEANS_ERR_STATE; } \
    } while (0)

// ------------------------------------------------------------------ layout
namespace {
struct Layout {
    size_t st, st_api, C, C32, Ca32, Chi, Clo, cn, cnimg, Ca, Cahi, Calo, cna, cnimga, C16h, C16l, Ca16h, Ca16l, lab0, lab1, flags, fb1, ftau, Xf, cand, cand_cnt, pair_rows, pair_j,
        scratch, packed1,
        upd_part, seg_bh, seg_off, seg_chunk, seg_cmap, xg_map, seed_d2, seed_near, seed_cc, seed_part, seed_T, seed_x, seed_idx, seed_u, perm, Gring, Fring, gram_part, trace,
        ub, lb, act_rows, pj2, pgap, C_ref, shift, ub0, lb0, pj20, pgap0, C_ref0, xchk, x2, sref, part0, part1, total,
        scratch_bytes;
    std::vector<size_t> guards;   // AAKM_WS_CANARY=1: a 256-B canary after every region
};

// Checked-workspace mode (compute-sanitizer is not available on the GPU pool): every
// workspace region is followed by a 256-byte canary filled at create; a kernel that
// writes past the end of its region changes it (kmeans_debug_check_canaries).
static bool ws_canary() {
    static const bool on = getenv("AAKM_WS_CANARY") && atoi(getenv("AAKM_WS_CANARY")) != 0;
    return on;
}
constexpr unsigned char CANARY = 0xA5;

size_t al(size_t x) { return (x + 255) & ~(size_t)255; }

// rows the tensor-core candidate refine can hold (more -> SIMT refine for the rest)
long long fcap_of(long long n) { return n / 4 + 4096; }

Layout layout(long long n, int d, int K, int m_max, bool bounded) {
    Layout L;
    size_t o = 0;
    const size_t KD = (size_t)K * d;
    const int H = m_max + 1;
    const bool canary = ws_canary();
    auto take = [&](size_t bytes) {
        size_t r = o;
        o = al(o + bytes);
        if (canary) { L.guards.push_back(o); o += 256; }
        return r;
    };
    L.st = take(sizeof(DevState));
    L.st_api = take(sizeof(DevState));
    L.C = take(KD * 8); L.C32 = take(KD * 4); L.Chi = take(KD * 4); L.Clo = take(KD * 4); L.cn = take((size_t)K * 4);
    const size_t cnimg = (size_t)((K + 127) / 128) * AAKM_CNIMG_BYTES;
    L.cnimg = take(cnimg);
    L.Ca = take(KD * 8); L.Ca32 = take(KD * 4); L.Cahi = take(KD * 4); L.Calo = take(KD * 4); L.cna = take((size_t)K * 4);
    L.cnimga = take(cnimg);
    L.C16h = take(KD * 2); L.C16l = take(KD * 2); L.Ca16h = take(KD * 2); L.Ca16l = take(KD * 2);
    L.lab0 = take((size_t)n * 4); L.lab1 = take((size_t)n * 4);
    L.flags = take((size_t)n * 4 + 4);
    const long long fc = fcap_of(n);
    L.fb1 = take((size_t)fc * 4 + 4);
    L.ftau = take((size_t)fc * 4 + 4);
    L.Xf = take((size_t)fc * d * 4 + 16);
    L.cand = take((size_t)fc * AAKM_MAXC * 4 + 4);
    L.cand_cnt = take((size_t)fc * 16 + 16);
    L.pair_rows = take((size_t)fc * 4 + 4);
    L.pair_j = take((size_t)fc * 8 + 8);
    const size_t pk = (2 * KD + K + 6) * 8;     // [S_hi | S_lo | N | E_hi | E_lo | E | changed | X2_hi | X2_lo] (pk_words)
    L.scratch = o;                         // one block, zeroed every pass: no canaries inside
    o = al(o + 256);                       // flag counts
    o = al(o + pk);                        // packed[0]
    L.packed1 = o;
    o = al(o + pk);                        // packed[1]
    L.scratch_bytes = o - L.scratch;
    if (canary) { L.guards.push_back(o); o += 256; }
    L.upd_part = take((size_t)AAKM_UPD_MAX_BLOCKS * 16);
    L.seg_bh = take((size_t)AAKM_SEG_BLOCKS_MAX * K * 4);
    L.seg_off = take((size_t)K * 4 + 4);
    L.seg_chunk = take((size_t)K * 4 + 4);
    L.seg_cmap = take(((size_t)n / 256 + K + 1) * 16);
    L.perm = take((size_t)n * 4 + 4);
    L.xg_map = take(128);
    L.seed_d2 = take((size_t)n * 8 + 16);           // + the 16-B tail of a bulk-copied odd run
    L.seed_near = take((size_t)n * 4);
    L.seed_cc = take((size_t)K * 8);
    L.seed_part = take((size_t)AAKM_SEED_BLOCKS * 8);
    L.seed_T = take((size_t)AAKM_MAX_RANKS * 8);
    L.seed_x = take((size_t)(d + 2) * 4);
    L.seed_idx = take((size_t)K * 8);
    L.seed_u = take((size_t)K * 8);
    L.Gring = take((size_t)H * KD * 8);             // fp64 Anderson history (R-A17)
    L.Fring = take((size_t)H * KD * 8);
    L.gram_part = take((size_t)AAKM_GRAM_BLOCKS * 2 * AAKM_H_SLOTS * 8);
    L.trace = take((size_t)AAKM_TRACE_CAP * sizeof(TraceRec));
    // bounded engine (2xFP16, cfg.bounded): 12 B per row + 2 centroid-sized arrays
    const size_t nb = bounded ? (size_t)n : 0;
    L.ub = take(nb * 4 + 4); L.lb = take(nb * 4 + 4); L.act_rows = take(nb * 4 + 4); L.pj2 = take(nb * 4 + 4);
    L.C_ref = take(bounded ? KD * 8 : 8); L.shift = take(bounded ? (size_t)K * 4 : 4);
    L.ub0 = take(nb * 4 + 4); L.lb0 = take(nb * 4 + 4); L.pj20 = take(nb * 4 + 4);
    L.pgap = take(nb * 4 + 4); L.pgap0 = take(nb * 4 + 4);
    L.C_ref0 = take(bounded ? KD * 8 : 8);
    L.xchk = take(16);
    L.x2 = take(16);
    L.sref = take((2 * KD + K) * 8);                // incremental update: S_hi | S_lo | N of P^{t-1}
    L.part0 = take(pk);                             // ... with a communicator: this rank's partials
    L.part1 = take(pk);                             //     (branch A / B; the allreduce's send buffers)
    L.total = o;
    return L;
}

kmeans_status validate(long long n_local, int d, int k, const kmeans_config* cfg, std::string& why) {
    if (!cfg) { why = "cfg is NULL"; return KMEANS_ERR_INVALID; }
    if (n_local < 0) { why = "n_local < 0"; return KMEANS_ERR_INVALID; }
    if (n_local > 0x7fffffffLL) { why = "n_local > 2^31-1 rows per rank"; return KMEANS_ERR_INVALID; }
    if (d < 1) { why = "d < 1"; return KMEANS_ERR_INVALID; }
    if (d > 4096) { why = "d > 4096 unsupported"; return KMEANS_ERR_INVALID; }
    if (k < 1) { why = "k < 1"; return KMEANS_ERR_INVALID; }
    if (cfg->m_max < 0 || cfg->m_max > KMEANS_M_MAX) { why = "m_max outside [0, 30]"; return KMEANS_ERR_INVALID; }
    if (cfg->m0 < 0 || cfg->m0 > cfg->m_max) { why = "m0 outside [0, m_max]"; return KMEANS_ERR_INVALID; }
    if (!(cfg->eps1 >= 0.0) || !(cfg->eps1 < cfg->eps2)) { why = "need 0 <= eps1 < eps2"; return KMEANS_ERR_INVALID; }
    if (cfg->max_iters < 1) { why = "max_iters < 1"; return KMEANS_ERR_INVALID; }
    if (!(cfg->ridge >= 0.0)) { why = "ridge < 0"; return KMEANS_ERR_INVALID; }
    if (cfg->assign_path < 0 || cfg->assign_path > 3) { why = "bad assign_path"; return KMEANS_ERR_INVALID; }
    if (cfg->assign_path == KMEANS_PATH_TC && !tc_supported(d, k)) {
        why = "tensor-core path needs d % 32 == 0 and d <= 128"; return KMEANS_ERR_INVALID;
    }
    if (cfg->assign_path == KMEANS_PATH_TC16 && !tc16_supported(d, k)) {
        why = "2xFP16 tensor-core path needs d in {64, 128}"; return KMEANS_ERR_INVALID;
    }
    return KMEANS_OK;
}
}  // namespace

// ------------------------------------------------------------------ enqueue helpers
static void assign_engine(kmeans_handle* h, const Dev& d, const GEval& g, cudaStream_t s) {
    if (d.ub) {                                   // bounded engine: Hamerly test, then the gathered rows
        h->launches += launch_bounds_prep(d, g, s);
        launch_assign_tc_bounded(d, g, d.st == h->d.st ? h->tcm : h->tcm_api, s);
    } else if (h->path == KMEANS_PATH_TC || h->path == KMEANS_PATH_TC16) {
        launch_assign_tc(d, g, d.st == h->d.st ? h->tcm : h->tcm_api, s);
    } else {
        launch_assign_simt(d, g, s);
    }
}

// Centroid prep after every change of C (a1 / a13): ||c||^2, tf32 split, and
// for the 2xFP16 engine the scaled fp16 hi/lo operands.
static void combine(kmeans_handle* h, const Dev& d, int mode, const double* src, cudaStream_t s) {
    launch_combine(d, mode, src, s);
    h->launches++;
    if (d.cnimg) { launch_csplit16(d, mode, s); h->launches++; }   // tensor operands (both kinds)
}

// Exact re-decision of the near-tie rows: the tensor-core engine re-runs the
// flagged rows in candidate mode (gather -> MMA pass -> fp64 on candidates);
// rows beyond the candidate capacity (and the SIMT engine) use the SIMT refine.
static void refine_engine(kmeans_handle* h, const Dev& d, const GEval& g, cudaStream_t s) {
    if (h->path == KMEANS_PATH_TC || h->path == KMEANS_PATH_TC16) {
        h->launches += launch_refine_tc(d, g, d.st == h->d.st ? h->tcm : h->tcm_api, s);
        h->launches += launch_refine(d, g, s, d.fcap);
    } else {
        h->launches += launch_refine(d, g, s, 0);
    }
}

// One integer allreduce of the packed partials: exact and order-free, so every
// rank (and every rank count) sees the same bytes.  The E slot is still zero
// here; k_energy fills it from the reduced sums afterwards.
// Out of place when the incremental update keeps this rank's partial (d.partial).
static kmeans_status allreduce(kmeans_handle* h, const Dev& d, int branch, cudaStream_t s) {
    if (!h->comm) return KMEANS_OK;                 // nranks == 1 (unless cfg.comm_always)
    const size_t cnt = (size_t)pk_words(h->d);     // the E slot is still 0 here (k_energy runs after)
    NK(h, ncclAllReduce(d.partial[branch], d.packed[branch], cnt, ncclInt64, ncclSum, h->comm, s));
    return KMEANS_OK;
}

// The assignment launch, bracketed by CUDA events on its own stream when timing
// (kmeans_assign_timing reads them back).
static kmeans_status timed_assign(kmeans_handle* h, const Dev& d, const GEval& g, cudaStream_t s, bool timing) {
    std::pair<cudaEvent_t, cudaEvent_t>* evp = nullptr;
    if (timing) {
        if (h->ev_used == h->ev.size()) {
            cudaEvent_t a, b;
            CK(h, cudaEventCreate(&a)); CK(h, cudaEventCreate(&b));
            h->ev.push_back({a, b});
        }
        evp = &h->ev[h->ev_used++];
        CK(h, cudaEventRecord(evp->first, s));
    }
    assign_engine(h, d, g, s);
    if (evp) CK(h, cudaEventRecord(evp->second, s));
    return KMEANS_OK;
}

// One G-evaluation (assign -> refine -> update partials -> allreduce -> control).
static kmeans_status geval(kmeans_handle* h, int branch, cudaStream_t s, bool timing) {
    Nvtx r0(branch == 0 ? "aakm:G-evaluation" : "aakm:G-evaluation (fallback)");
    const Dev& d = h->d;
    GEval g{};
    g.branch = branch; g.force = 0; g.prev_mode = 0;
    if (branch == 1) { combine(h, d, 1, nullptr, s); dbg("combine_fb", s); }
    kmeans_status st = KMEANS_OK;
    NvtxStep step;
    step.to("aakm:assign");                                 // Eq. 3: contraction + argmin + refine
    if (branch == 0 && h->feed_chunks > 0) {                // streamed X: each row chunk once it landed
        const long long T = (d.n + 127) / 128;
        for (int c = 0; c < h->feed_chunks; ++c) {
            CK(h, cudaStreamWaitEvent(s, h->feed_ev[c], 0));
            GEval gc = g;
            gc.tile0 = c * h->feed_tiles;
            gc.tile1 = std::min(T, (c + 1) * h->feed_tiles);
            launch_assign_tc(d, gc, h->tcm, s);
        }
        h->launches += h->feed_chunks - 1;
    } else {
        st = timed_assign(h, d, g, s, timing && branch == 0);
    }
    if (st != KMEANS_OK) return st;
    dbg("assign", s);
    refine_engine(h, d, g, s);
    dbg("refine", s);
    step.to("aakm:update");                                 // Eq. 4: partial sums S, N (+ combine)
    std::pair<cudaEvent_t, cudaEvent_t>* uevp = nullptr;
    if (timing && branch == 0) {
        if (h->uev_used == h->uev.size()) {
            cudaEvent_t a, b;
            CK(h, cudaEventCreate(&a)); CK(h, cudaEventCreate(&b));
            h->uev.push_back({a, b});
        }
        uevp = &h->uev[h->uev_used++];
        CK(h, cudaEventRecord(uevp->first, s));
    }
    if (branch == 0 && h->feed_chunks > 0)                 // streamed X: the update reads every row and X2
        CK(h, cudaStreamWaitEvent(s, h->feed_all, 0));
    if (d.fused) h->launches += launch_fused_zero(d, g, h->fused, s);      // f4: zero + "zeroed" barrier
    h->launches += 1 + launch_update(d, g, s);       // + the assignment launch
    if (uevp) CK(h, cudaEventRecord(uevp->second, s));
    dbg("update", s);
    if (d.fused) {
        h->launches += launch_fused_flushed(d, g, h->fused, s);           // f4: "flushed" barrier
    } else {
        st = allreduce(h, d, branch, s);
        if (st != KMEANS_OK) return st;
    }
    if (h->comm) dbg("combine", s);
    step.to("aakm:energy+control");                         // Eq. 1 and Algorithm 1's rules
    h->launches += launch_energy_x(d, g, s);        // sorted engine: E's parts from X2, N, S, C
    launch_control(d, branch, s);                   // E from the reduced parts + Algorithm 1 control
    dbg("control", s);
    h->launches += 1;
    return KMEANS_OK;
}

// One loop pass of Algorithm 1 (also used for line 1 when init_mode is set).
static kmeans_status enqueue_pass(kmeans_handle* h, cudaStream_t s, bool timing) {
    Nvtx r0("aakm:pass");
    const Dev& d = h->d;
    CK(h, cudaMemsetAsync(h->scratch, 0, h->scratch_bytes, s));
    if (d.partial[0] != d.packed[0]) {                    // this rank's local partials (both branches)
        const size_t pkb = (size_t)pk_words(d) * 8;
        CK(h, cudaMemsetAsync(d.partial[0], 0, pkb, s));
        CK(h, cudaMemsetAsync(d.partial[1], 0, pkb, s));
    }
    dbg("memset", s);
    kmeans_status st = geval(h, 0, s, timing);
    if (st != KMEANS_OK) return st;
    if (d.condB) {
        // graph capture: the fallback G-evaluation (branch B) goes into the body of a
        // conditional IF node that k_control switches on only for a rejected iterate,
        // so a pass without a rejection launches none of its ~10 kernels
        cudaStreamCaptureStatus cst;
        cudaGraph_t g;
        const cudaGraphNode_t* deps = nullptr;
        size_t nd = 0;
        CK(h, cudaStreamGetCaptureInfo(s, &cst, nullptr, &g, &deps, &nd));
        alignas(cudaGraphNodeParams) unsigned char praw[sizeof(cudaGraphNodeParams)] = {};   // (a union: no default ctor)
        cudaGraphNodeParams& p = *reinterpret_cast<cudaGraphNodeParams*>(praw);
        p.type = cudaGraphNodeTypeConditional;
        p.conditional.handle = d.condB;
        p.conditional.type = cudaGraphCondTypeIf;
        p.conditional.size = 1;
        cudaGraphNode_t node;
        CK(h, cudaGraphAddNode(&node, g, deps, nd, &p));
        if (!h->body_stream) CK(h, cudaStreamCreateWithFlags(&h->body_stream, cudaStreamNonBlocking));
        CK(h, cudaStreamBeginCaptureToGraph(h->body_stream, p.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                            cudaStreamCaptureModeThreadLocal));
        const long long b0 = h->launches;
        st = geval(h, 1, h->body_stream, false);
        cudaGraph_t body;
        const cudaError_t e = cudaStreamEndCapture(h->body_stream, &body);
        if (st != KMEANS_OK) return st;
        CK(h, e);
        h->kernels_b = h->launches - b0;
        CK(h, cudaStreamUpdateCaptureDependencies(s, &node, 1, cudaStreamSetCaptureDependencies));
    } else {
        st = geval(h, 1, s, false);
        if (st != KMEANS_OK) return st;
    }
    Nvtx r2("aakm:anderson");                               // Eq. 6-8: G, F, Gram, solve, mix
    launch_finalize(d, s);
    dbg("finalize", s);
    launch_gram(d, s);
    dbg("gram", s);
    launch_solve(d, s);
    dbg("solve", s);
    combine(h, d, 0, nullptr, s);
    dbg("combine_mix", s);
    launch_advance(d, s);
    dbg("advance", s);
    h->launches += 4;                               // finalize, gram, gram_reduce + solve (one launch), advance
    CK(h, cudaGetLastError());
    return KMEANS_OK;
}

static kmeans_status ensure_graph(kmeans_handle* h) {
    if (h->pass_exec) return KMEANS_OK;
    // The caller's stream may be the legacy NULL stream (torch's default), which
    // cannot be captured: capture on a private stream, replay on the caller's.
    cudaGraph_t g;
    long long before = h->launches;
    CK(h, cudaStreamBeginCapture(h->cap_stream, cudaStreamCaptureModeThreadLocal));
    // branch B as a conditional node (not with a plain NCCL communicator: its captured
    // collectives stay outside conditional bodies; the predicated kernels run instead)
    h->kernels_b = 0;
    // (tiny shards keep the predicated kernels: c1's 50-us passes ran 10 % slower with
    // the conditional node, c2's Lloyd passes 9 % faster, c3 1-4 %)
    if ((!h->comm || h->d.fused) && h->n_global >= 50000) {
        cudaStreamCaptureStatus cst;
        cudaGraph_t cg;
        CK(h, cudaStreamGetCaptureInfo(h->cap_stream, &cst, nullptr, &cg, nullptr, nullptr));
        cudaGraphConditionalHandle hb;
        CK(h, cudaGraphConditionalHandleCreate(&hb, cg, 0, cudaGraphCondAssignDefault));
        h->d.condB = hb;
    }
    kmeans_status st = enqueue_pass(h, h->cap_stream, false);
    h->d.condB = 0;                                 // eager launches never touch the handle
    cudaError_t e = cudaStreamEndCapture(h->cap_stream, &g);
    if (st != KMEANS_OK) return st;
    CK(h, e);
    CK(h, cudaGraphInstantiate(&h->pass_exec, g, 0));
    CK(h, cudaGraphDestroy(g));
    h->kernels_per_pass = h->launches - before;
    h->launches = before;
    return KMEANS_OK;
}

static kmeans_status start(kmeans_handle* h, const double* C0) {
    launch_reset(h->d, h->stream);
    dbg("reset", h->stream);
    combine(h, h->d, 2, C0, h->stream);
    dbg("combine_c0", h->stream);
    h->launches += 2;
    return enqueue_pass(h, h->stream, h->cfg.timing != 0);   // Algorithm 1 line 1
}

// Every resource a handle may hold, released in one place (kmeans_destroy and
// every failure exit of kmeans_create).  sync: drain the streams first.
static void release(kmeans_handle* h, bool sync) {
    if (!h) return;
    if (sync && h->stream) cudaStreamSynchronize(h->stream);
    if (h->pass_exec) cudaGraphExecDestroy(h->pass_exec);
    if (h->cap_stream) cudaStreamDestroy(h->cap_stream);
    if (h->body_stream) cudaStreamDestroy(h->body_stream);
    if (h->copy_stream) {
        if (sync) cudaStreamSynchronize(h->copy_stream);
        cudaStreamDestroy(h->copy_stream);
        for (auto e : h->feed_ev) if (e) cudaEventDestroy(e);
        if (h->feed_gate) cudaEventDestroy(h->feed_gate);
        if (h->feed_all) cudaEventDestroy(h->feed_all);
    }
    if (h->tcm) tc_free_maps(h->tcm);
    if (h->tcm_api) tc_free_maps(h->tcm_api);
    for (auto& e : h->ev) { cudaEventDestroy(e.first); cudaEventDestroy(e.second); }
    for (auto& e : h->uev) { cudaEventDestroy(e.first); cudaEventDestroy(e.second); }
    if (h->run_ev[0]) cudaEventDestroy(h->run_ev[0]);
    if (h->run_ev[1]) cudaEventDestroy(h->run_ev[1]);
    if (h->sync_ev) cudaEventDestroy(h->sync_ev);
    if (h->st_host) cudaFreeHost(h->st_host);
    if (h->tr_host) cudaFreeHost(h->tr_host);
    if (h->scal_host) cudaFreeHost(h->scal_host);
    if (h->done_host) cudaFreeHost(h->done_host);
    if (h->fused) fused_free(h->fused, h->comm);
    if (h->comm) {
        if (sync) ncclCommDestroy(h->comm);
        else ncclCommAbort(h->comm);             // a failed / poisoned communicator may never complete
    }
    delete h;
}

static double comm_timeout_s() {
    static const double t = getenv("AAKM_COMM_TIMEOUT_S") ? atof(getenv("AAKM_COMM_TIMEOUT_S")) : 600.0;
    return t > 0.0 ? t : 600.0;
}

static kmeans_status sync_stream(kmeans_handle* h, cudaStream_t s) {
    if (!h->comm) {
        CK(h, cudaStreamSynchronize(s));
        return KMEANS_OK;
    }
    if (!h->sync_ev) CK(h, cudaEventCreateWithFlags(&h->sync_ev, cudaEventDisableTiming));
    CK(h, cudaEventRecord(h->sync_ev, s));
    const auto t0 = std::chrono::steady_clock::now();
    for (unsigned spin = 0;; ++spin) {
        const cudaError_t q = cudaEventQuery(h->sync_ev);
        if (q == cudaSuccess) return KMEANS_OK;
        if (q != cudaErrorNotReady) CK(h, q);
        ncclResult_t ar = ncclSuccess;
        ncclResult_t r = ncclCommGetAsyncError(h->comm, &ar);
        if (r != ncclSuccess || (ar != ncclSuccess && ar != ncclInProgress)) {
            h->err = std::string("NCCL asynchronous error: ") + ncclGetErrorString(r != ncclSuccess ? r : ar);
            ncclCommAbort(h->comm);
            h->comm = nullptr;
            h->poisoned = true;
            return KMEANS_ERR_NCCL;
        }
        const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (el > comm_timeout_s()) {
            h->err = "collective did not complete within AAKM_COMM_TIMEOUT_S seconds (peer failure?): communicator aborted";
            ncclCommAbort(h->comm);
            h->comm = nullptr;
            h->poisoned = true;
            return KMEANS_ERR_NCCL;
        }
        if (spin > 64) std::this_thread::sleep_for(std::chrono::microseconds(50));
    }
}

// kmeans_aa_step_host refreshed X with rows outside the create-time ranges: the
// pass that used them is meaningless, so the handle is poisoned.
static void x_range_error(kmeans_handle* h) {
    h->err = "X_host rows exceed the create-time range of X (max |x_ik| or max ||x_i||): "
             "every operand and fixed-point scale was derived from it";
    h->poisoned = true;
}

// One-time kernel attribute setup (max dynamic shared memory) PER DEVICE: the
// attributes are device state, so a handle on a second GPU repeats it.
namespace aakm { int g_pdl = [] { const char* v = getenv("AAKM_PDL"); return v ? atoi(v) : 1; }(); }

static cudaError_t setup_device(int dev) {
    static std::mutex mu;
    static bool done[AAKM_MAX_DEVICES] = {};
    if (dev < 0 || dev >= AAKM_MAX_DEVICES) return cudaErrorInvalidDevice;
    std::lock_guard<std::mutex> lk(mu);
    if (done[dev]) return cudaSuccess;
    for (cudaError_t e : {setup_simt(), setup_refine(), setup_update(), setup_tc(), setup_seed()})
        if (e != cudaSuccess) return e;
    done[dev] = true;
    return cudaSuccess;
}

// ------------------------------------------------------------------ ABI
extern "C" {

int32_t kmeans_abi_version(void) { return KMEANS_ABI_VERSION; }

kmeans_status kmeans_config_default(kmeans_config* cfg) {
    if (!cfg) return KMEANS_ERR_INVALID;
    memset(cfg, 0, sizeof(*cfg));
    cfg->m0 = 2; cfg->m_max = 30; cfg->eps1 = 0.02; cfg->eps2 = 0.5;
    cfg->dynamic_m = 1; cfg->max_iters = 10000; cfg->ridge = 1e-10;
    cfg->assign_path = KMEANS_PATH_AUTO; cfg->timing = 0; cfg->bounded = 0;
    return KMEANS_OK;
}

kmeans_status kmeans_workspace_size(int64_t n_local, int32_t d, int32_t k, const kmeans_config* cfg,
                                    size_t* bytes) {
    std::string why;
    if (!bytes) return KMEANS_ERR_INVALID;
    kmeans_status s = validate(n_local, d, k, cfg, why);
    if (s != KMEANS_OK) { g_create_err = why; return s; }
    *bytes = layout(n_local, d, k, cfg->m_max, cfg->bounded != 0).total;
    return KMEANS_OK;
}

kmeans_status kmeans_nccl_unique_id(void* uid128) {
    if (!uid128) return KMEANS_ERR_INVALID;
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess) { g_create_err = "ncclGetUniqueId failed"; return KMEANS_ERR_NCCL; }
    static_assert(sizeof(ncclUniqueId) == 128, "nccl id size");
    memcpy(uid128, &id, 128);
    return KMEANS_OK;
}

kmeans_status kmeans_create(kmeans_handle** out, const float* X, int64_t n_local, int64_t n_global,
                            int32_t d, int32_t k, const kmeans_config* cfg, void* workspace,
                            size_t workspace_bytes, int32_t rank, int32_t nranks, const void* uid128,
                            kmeans_stream_t stream) {
    Nvtx nvtx_("kmeans_create");
    std::string why;
    if (!out) { g_create_err = "out is NULL"; return KMEANS_ERR_INVALID; }
    *out = nullptr;
    kmeans_status vs = validate(n_local, d, k, cfg, why);
    if (vs != KMEANS_OK) { g_create_err = why; return vs; }
    if ((!X && n_local > 0) || !workspace) { g_create_err = "X or workspace is NULL"; return KMEANS_ERR_INVALID; }
    if (nranks < 1 || nranks > AAKM_MAX_RANKS || rank < 0 || rank >= nranks) { g_create_err = "bad rank/nranks"; return KMEANS_ERR_INVALID; }
    if ((nranks == 1) != (uid128 == nullptr)) { g_create_err = "uid128 must be NULL iff nranks == 1"; return KMEANS_ERR_INVALID; }
    if (n_global < n_local || k > n_global) { g_create_err = "need n_local <= n_global and k <= n_global"; return KMEANS_ERR_INVALID; }
    if (((uintptr_t)workspace & 255) != 0) { g_create_err = "workspace must be 256-byte aligned"; return KMEANS_ERR_INVALID; }
    Layout L = layout(n_local, d, k, cfg->m_max, cfg->bounded != 0);
    if (workspace_bytes < L.total) { g_create_err = "workspace too small"; return KMEANS_ERR_INVALID; }

    kmeans_handle* h = new kmeans_handle();
    h->cfg = *cfg;
    h->stream = (cudaStream_t)stream;
    h->rank = rank; h->nranks = nranks; h->n_global = n_global;
    // AUTO: 2xFP16 tensor engine for d in {64, 128} (same rigorous bound + exact refine as
    // 3xTF32, 1.4x its throughput on B200), 3xTF32 for other d % 32 == 0, else FP32 SIMT.
    h->path = cfg->assign_path != KMEANS_PATH_AUTO ? cfg->assign_path
            : tc16_supported(d, k) ? KMEANS_PATH_TC16
            : tc_supported(d, k) ? KMEANS_PATH_TC : KMEANS_PATH_SIMT;
    char* w = (char*)workspace;
    Dev& D = h->d;
    memset(&D, 0, sizeof(D));
    D.X = X; D.n = n_local; D.d = d; D.K = k; D.H = cfg->m_max + 1; D.m_max = cfg->m_max; D.m0 = cfg->m0;
    D.dynamic_m = cfg->dynamic_m; D.max_iters = cfg->max_iters; D.eps1 = cfg->eps1; D.eps2 = cfg->eps2;
    D.ridge = cfg->ridge;
    D.st = (DevState*)(w + L.st);
    D.C = (double*)(w + L.C); D.C32 = (float*)(w + L.C32); D.Chi = (float*)(w + L.Chi); D.Clo = (float*)(w + L.Clo); D.cn = (float*)(w + L.cn);
    D.lab[0] = (int*)(w + L.lab0); D.lab[1] = (int*)(w + L.lab1);
    D.flag_rows = (int*)(w + L.flags);
    D.flag_b1 = (float*)(w + L.fb1);
    D.flag_tau = (float*)(w + L.ftau);
    D.Xf = (float*)(w + L.Xf);
    D.cand = (int*)(w + L.cand);
    D.cand_cnt = (int*)(w + L.cand_cnt);
    D.fcap = fcap_of(n_local);
    D.flag_count = (long long*)(w + L.scratch);
    D.act_count = (long long*)(w + L.scratch + 32);                   // [2], zeroed per pass with the flags
    D.pair_count = (long long*)(w + L.scratch + 64);                  // [2], likewise
    D.delta_count = (long long*)(w + L.scratch + 96);                 // [2], likewise
    D.pair_rows = (int*)(w + L.pair_rows); D.pair_j = (int2*)(w + L.pair_j);
    D.packed[0] = (long long*)(w + L.scratch + 256);
    D.packed[1] = (long long*)(w + L.packed1);
    D.partial[0] = D.packed[0]; D.partial[1] = D.packed[1];          // local buffers: below, if used
    D.upd_part = (double*)(w + L.upd_part);
    D.seg_bh = (int*)(w + L.seg_bh);
    D.seg_off = (int*)(w + L.seg_off);
    D.seg_chunk = (int*)(w + L.seg_chunk);
    D.seg_cmap = (int4*)(w + L.seg_cmap);
    D.seed_d2 = (long long*)(w + L.seed_d2); D.seed_part = (long long*)(w + L.seed_part);
    D.seed_near = (int*)(w + L.seed_near); D.seed_cc = (double*)(w + L.seed_cc);
    D.seed_T = (long long*)(w + L.seed_T); D.seed_x = (int*)(w + L.seed_x);
    D.seed_idx = (long long*)(w + L.seed_idx); D.seed_u = (double*)(w + L.seed_u);
    D.perm = (int*)(w + L.perm);
    D.Gring = (double*)(w + L.Gring); D.Fring = (double*)(w + L.Fring);
    D.gram_part = (double*)(w + L.gram_part);
    D.trace = (TraceRec*)(w + L.trace);
    D.nranks = nranks;
    {
        long long KD = (long long)k * d;
        long long ub = (n_local + 255) / 256;
        if (ub > AAKM_UPD_MAX_BLOCKS) ub = AAKM_UPD_MAX_BLOCKS;
        D.upd_blocks = (int)(ub < 1 ? 1 : ub);
        long long gb = (KD + 127) / 128;
        D.gram_blocks = (int)(gb > AAKM_GRAM_BLOCKS ? AAKM_GRAM_BLOCKS : (gb < 1 ? 1 : gb));
    }
    D.tc_kind = h->path == KMEANS_PATH_TC16 ? 1 : 0;
    D.pair_ok = (h->path == KMEANS_PATH_TC16 || h->path == KMEANS_PATH_TC) && (d == 32 || d == 64 || d == 128);
    const bool tcpath = h->path == KMEANS_PATH_TC || h->path == KMEANS_PATH_TC16;
    D.cnimg = tcpath ? (uint8_t*)(w + L.cnimg) : nullptr;
    D.key_mul = 32u;
    if (h->path == KMEANS_PATH_TC16 && cfg->bounded) {                 // bounded engine (Algorithm 1 passes)
        D.ub = (float*)(w + L.ub); D.lb = (float*)(w + L.lb); D.act_rows = (int*)(w + L.act_rows);
        D.pj2 = (int*)(w + L.pj2);
        D.C_ref = (double*)(w + L.C_ref); D.shift = (float*)(w + L.shift);
        D.ub0 = (float*)(w + L.ub0); D.lb0 = (float*)(w + L.lb0); D.pj20 = (int*)(w + L.pj20);
        D.C_ref0 = (double*)(w + L.C_ref0);
        if (!getenv("AAKM_NO_PGAP")) { D.pgap = (float*)(w + L.pgap); D.pgap0 = (float*)(w + L.pgap0); }
    }
    D.dbg = getenv("AAKM_TC_DBG") ? atoi(getenv("AAKM_TC_DBG")) : 0;
    if (getenv("AAKM_TC_TRACE")) {                                     // perf probe only: a 32 KB stamp buffer
        if (cudaMalloc(&D.dbg_ts, (2 * 8 * 256 + 256) * 8) != cudaSuccess) D.dbg_ts = nullptr;
        else cudaMemset(D.dbg_ts, 0, (2 * 8 * 256 + 256) * 8);
    }
    D.Chi16 = w + L.C16h; D.Clo16 = w + L.C16l;
    D.x_scale = 1.f; D.x_inv_scale = 1.f; D.x_absmax = 0.f;
    D.tau_gamma = h->path == KMEANS_PATH_TC ? tau_gamma_tc(d)
                : h->path == KMEANS_PATH_TC16 ? tau_gamma_tc16(d) : tau_gamma_simt(d);
    h->da = D;
    h->da.ub = nullptr; h->da.lb = nullptr; h->da.act_rows = nullptr;    // the API calls stay dense
    h->da.pj2 = nullptr;
    h->da.C_ref = nullptr; h->da.shift = nullptr;
    h->da.ub0 = nullptr; h->da.lb0 = nullptr; h->da.pj20 = nullptr; h->da.C_ref0 = nullptr;
    h->da.pgap = nullptr; h->da.pgap0 = nullptr;
    h->da.st = (DevState*)(w + L.st_api);
    h->da.C = (double*)(w + L.Ca); h->da.C32 = (float*)(w + L.Ca32); h->da.Chi = (float*)(w + L.Cahi); h->da.Clo = (float*)(w + L.Calo);
    h->da.cn = (float*)(w + L.cna);
    h->da.cnimg = tcpath ? (uint8_t*)(w + L.cnimga) : nullptr;
    h->da.Chi16 = w + L.Ca16h; h->da.Clo16 = w + L.Ca16l;
    h->scratch = w + L.scratch;
    h->scratch_bytes = L.scratch_bytes;
    h->xchk = (unsigned int*)(w + L.xchk);
    h->guards = L.guards;
    h->ws_base = w;

#define CKC(call)                                                                         \
    do {                                                                                  \
        cudaError_t e_ = (call);                                                          \
        if (e_ != cudaSuccess) {                                                          \
            g_create_err = std::string(#call) + ": " + cudaGetErrorString(e_);            \
            release(h, false);                                                            \
            return KMEANS_ERR_CUDA;                                                       \
        }                                                                                 \
    } while (0)
    CKC(cudaGetDevice(&D.dev));
    CKC(cudaDeviceGetAttribute(&D.num_sms, cudaDevAttrMultiProcessorCount, D.dev));
    D.seg_blocks = seg_blocks_for(k, D.num_sms);
    h->da.dev = D.dev; h->da.num_sms = D.num_sms; h->da.seg_blocks = D.seg_blocks;
    CKC(setup_device(D.dev));
    CKC(cudaStreamCreateWithFlags(&h->cap_stream, cudaStreamNonBlocking));
    // this rank's max |x_ik| and max ||x_i||^2 (one pass; float bits of non-negative
    // values order as uints): the 2xFP16 operand scale (rank-local) and, reduced
    // over the ranks below, the scales of the exact update sums
    float mloc[2] = {0.f, 0.f};
    {
        unsigned int* mx = (unsigned int*)(w + L.scratch);
        CKC(cudaMemsetAsync(mx, 0, 8, h->stream));
        launch_xstats_max(X, n_local, d, mx, h->stream);
        CKC(cudaMemcpyAsync(mloc, mx, 8, cudaMemcpyDeviceToHost, h->stream));
        CKC(cudaStreamSynchronize(h->stream));
        memcpy(h->x_stat, mloc, 8);
    }
    if (h->path == KMEANS_PATH_TC16 || h->path == KMEANS_PATH_TC) {   // common operand scale s (window keys)
        const float m = mloc[0];
        const float sx = m > 0.f ? exp2f(ceilf(log2f(m)) - 13.0f) : 1.0f;
        const float xnm = sqrtf(mloc[1]) * (1.0f + 1e-6f);   // (already rounded up in fp32) margin
        for (Dev* dv : {&h->d, &h->da}) {
            dv->x_absmax = m; dv->x_scale = sx; dv->x_inv_scale = 1.0f / sx; dv->x_nmax = xnm;
        }
    }
    if (h->path == KMEANS_PATH_TC || h->path == KMEANS_PATH_TC16) {
        h->tcm = tc_make_maps(h->d);
        h->tcm_api = tc_make_maps(h->da);
        if (!h->tcm || !h->tcm_api) {
            g_create_err = "cuTensorMapEncodeTiled failed for the tensor-core engine";
            release(h, false);
            return KMEANS_ERR_CUDA;
        }
    }
    {   // gather4 map of X for the update's segmented sums (generic kernel if unavailable)
        alignas(64) unsigned char map[128];
        const int lpr = d / 4;
        if (d % 4 == 0 && lpr <= 32 && (lpr & (lpr - 1)) == 0 && encode_gather_rows(map, X, n_local, d)) {
            CKC(cudaMemcpyAsync(w + L.xg_map, map, 128, cudaMemcpyHostToDevice, h->stream));
            CKC(cudaStreamSynchronize(h->stream));
            h->d.xg_map = w + L.xg_map; h->da.xg_map = w + L.xg_map;
        }
    }
    CKC(cudaMallocHost(&h->st_host, sizeof(DevState)));
    CKC(cudaMallocHost(&h->tr_host, sizeof(TraceRec) * 2));
    CKC(cudaMallocHost(&h->scal_host, 64));
    CKC(cudaMallocHost(&h->done_host, 64));
    CKC(cudaEventCreate(&h->run_ev[0]));
    CKC(cudaEventCreate(&h->run_ev[1]));
    for (size_t g : L.guards) CKC(cudaMemsetAsync(w + g, CANARY, 256, h->stream));
    CKC(cudaMemsetAsync(w + L.st, 0, sizeof(DevState), h->stream));
    CKC(cudaMemsetAsync(w + L.st_api, 0, sizeof(DevState), h->stream));
    CKC(cudaMemsetAsync(w + L.upd_part, 0, (size_t)AAKM_UPD_MAX_BLOCKS * 16, h->stream));
    if (nranks > 1 || cfg->comm_always) {
        // nranks == 1 with cfg.comm_always: a real 1-rank communicator, so every
        // allreduce of the data plane runs through NCCL (tests of that path on one GPU)
        ncclUniqueId id;
        if (nranks > 1) memcpy(&id, uid128, 128);
        else if (ncclGetUniqueId(&id) != ncclSuccess) { g_create_err = "ncclGetUniqueId failed"; release(h, false); return KMEANS_ERR_NCCL; }
        ncclResult_t r = ncclCommInitRank(&h->comm, nranks, id, rank);
        if (r != ncclSuccess) {
            h->comm = nullptr;
            g_create_err = std::string("ncclCommInitRank: ") + ncclGetErrorString(r);
            release(h, false);
            return KMEANS_ERR_NCCL;
        }
    }
    // Scales of the exact fixed-point update and energy sums (update.cu), from
    // statistics of X over ALL ranks, so every rank forms identical bytes.
    {
        unsigned int* mx = (unsigned int*)(w + L.scratch);            // scratch is free until the first pass
        CKC(cudaMemcpyAsync(mx, mloc, 8, cudaMemcpyHostToDevice, h->stream));
        if (h->comm) {
            ncclResult_t r = ncclAllReduce(mx, mx, 2, ncclFloat32, ncclMax, h->comm, h->stream);
            if (r != ncclSuccess) { g_create_err = std::string("ncclAllReduce: ") + ncclGetErrorString(r); release(h, false); return KMEANS_ERR_NCCL; }
        }
        unsigned int mb[2];
        CKC(cudaMemcpyAsync(mb, mx, 8, cudaMemcpyDeviceToHost, h->stream));
        if (sync_stream(h, h->stream) != KMEANS_OK) {           // polls NCCL errors / timeout
            g_create_err = h->err;
            release(h, false);
            return KMEANS_ERR_NCCL;
        }
        float mf[2];
        memcpy(mf, mb, 8);
        int ex = 0;
        if (mf[0] > 0.f) frexpf(mf[0], &ex);                           // max |x| < 2^ex
        const bool srt = update_sorted(n_global, d, k);
        // sorted engine energy (k_energy_x): sum_i ||x_i||^2 in units 2^x2_e, the finest
        // grid any pass's energy_q can ask for (B >= 2 xn_gmax^2, the cm = 0 case)
        const double xg = sqrt((double)mf[1]) * (1.0 + 1e-6);
        const double B0 = 2.0 * (xg + 0.0) * (xg + 0.0);
        int eb0 = 0;
        frexp(B0 > 0.0 ? B0 : 1.0, &eb0);
        for (Dev* dv : {&h->d, &h->da}) {
            dv->fx_scale = ldexpf(1.0f, 22 - ex);
            dv->fx_inv = ldexp(1.0, ex - 22);
            dv->xn_gmax = xg;                                          // max_i ||x_i||, rounded up
            dv->upd_sorted = srt ? 1 : 0;
            // one-kernel update for small K*d shards (AAKM_UPD_PRIV=0 forces the sort path)
            dv->upd_priv = srt && (long long)k * d <= AAKM_PRIV_MAX_KD && d <= 64 && n_local <= AAKM_PRIV_MAX_ROWS &&
                           !(getenv("AAKM_UPD_PRIV") && atoi(getenv("AAKM_UPD_PRIV")) == 0);
            dv->x2_e = eb0 - 51;
            dv->x2 = srt ? (long long*)(w + L.x2) : nullptr;
        }
        // incremental update (update.cu k_delta_*): the sorted engine and the plain combine;
        // S_ref is this rank's own partial (with a communicator the update adds into local
        // buffers and the allreduce reads them out of place); AAKM_DELTA_DIV: moved-row
        // threshold n_local / DIV (0: off)
        {
            const char* dv = getenv("AAKM_DELTA_DIV");
            const long long div = dv ? atoll(dv) : 64;
            const bool on = srt && !h->d.upd_priv && !cfg->fused_comm && div > 0;
            h->d.sref = on ? (long long*)(w + L.sref) : nullptr;
            h->d.delta_max = on ? n_local / div : 0;
            h->da.sref = nullptr; h->da.delta_max = 0;                 // API calls: always the full update
            if (on && h->comm) {                                       // S_ref must be this rank's own sums:
                h->d.partial[0] = (long long*)(w + L.part0);          // the update adds into local buffers,
                h->d.partial[1] = (long long*)(w + L.part1);          // the allreduce reads them out of place
            }
        }
        if (srt) {
            CKC(cudaMemsetAsync(w + L.x2, 0, 16, h->stream));
            launch_x2(X, n_local * d, eb0 - 51, (long long*)(w + L.x2), h->stream);
        }
        h->x_gamax = mf[0];
        if (cfg->fused_comm) {                                         // f4: packed vectors in a symmetric window
            const char* m = h->comm ? fused_setup(&h->fused, h->comm, h->d, w + L.scratch, h->stream)
                                    : "fused_comm needs a communicator (nranks > 1 or comm_always)";
            if (m) {
                g_create_err = m;
                release(h, false);
                return h->comm ? KMEANS_ERR_NCCL : KMEANS_ERR_INVALID;
            }
        }
        CKC(cudaMemsetAsync(w + L.scratch, 0, 128, h->stream));
    }
    CKC(cudaStreamSynchronize(h->stream));
#undef CKC
    *out = h;
    return KMEANS_OK;
}

kmeans_status kmeans_assign(kmeans_handle* h, const double* C, const int32_t* labels_prev, int32_t* labels_out,
                            double* energy_out, int64_t* changed_out) {
    Nvtx nvtx_("kmeans_assign");
    LIVE(h);
    if (!C || (!labels_out && h->d.n > 0)) FAIL(h, KMEANS_ERR_INVALID, "C or labels_out is NULL");
    cudaStream_t s = h->stream;
    const Dev& d = h->da;
    CK(h, cudaMemsetAsync(h->scratch, 0, h->scratch_bytes, s));
    combine(h, d, 2, C, s);
    GEval g{};
    g.branch = 0; g.force = 1; g.lab_out = labels_out;
    g.prev_mode = labels_prev ? 2 : 1; g.lab_prev = labels_prev;
    kmeans_status st = timed_assign(h, d, g, s, h->cfg.timing != 0);
    if (st != KMEANS_OK) return st;
    refine_engine(h, d, g, s);
    h->launches += 1 + launch_update(d, g, s);       // + the assignment launch
    st = allreduce(h, d, 0, s);
    if (st != KMEANS_OK) return st;
    h->launches += launch_energy_x(d, g, s);
    launch_energy(d, g, s);
    h->launches += 1;
    CK(h, cudaMemcpyAsync(h->scal_host, d.packed[0] + pk_e(d), 16, cudaMemcpyDeviceToHost, s));   // E, changed
    CK(h, cudaMemcpyAsync(h->scal_host + 2, d.flag_count, 8, cudaMemcpyDeviceToHost, s));
    SYNC(h, s);
    CK(h, cudaGetLastError());
    long long raw[2];
    memcpy(raw, h->scal_host, 16);
    if (energy_out) memcpy(energy_out, &raw[0], 8);                  // fp64 bits (k_energy)
    if (changed_out) *changed_out = labels_prev ? (int64_t)raw[1] : 0;
    return KMEANS_OK;
}

kmeans_status kmeans_debug_scores(kmeans_handle* h, const double* C, float* rows_out, int32_t* kind_out,
                                  double* unit_out) {
    LIVE(h);
    if (!C || (!rows_out && h->d.n > 0) || !kind_out || !unit_out) FAIL(h, KMEANS_ERR_INVALID, "NULL argument");
    cudaStream_t s = h->stream;
    Dev d = h->da;
    d.dbg_rows = reinterpret_cast<float4*>(rows_out);
    CK(h, cudaMemsetAsync(h->scratch, 0, h->scratch_bytes, s));
    combine(h, d, 2, C, s);
    GEval g{};
    g.branch = 0; g.force = 1; g.lab_out = d.lab[0]; g.prev_mode = 1;
    assign_engine(h, d, g, s);
    h->launches += 1;
    float sc = 1.f;
    CK(h, cudaMemcpyAsync(h->scal_host, &d.st->c_scale, 4, cudaMemcpyDeviceToHost, s));
    SYNC(h, s);
    CK(h, cudaGetLastError());
    memcpy(&sc, h->scal_host, 4);
    if (h->path == KMEANS_PATH_TC16 || h->path == KMEANS_PATH_TC) { *kind_out = 1; *unit_out = 0.5 / ((double)sc * (double)sc); }
    else { *kind_out = 2; *unit_out = 1.0; }
    return KMEANS_OK;
}

kmeans_status kmeans_bounds_export(kmeans_handle* h, float* ub_out, float* lb_out, int32_t* p2_out, double* Cref_out) {
    LIVE(h);
    const Dev& d = h->d;
    if (!d.ub) FAIL(h, KMEANS_ERR_INVALID, "handle has no bounded engine (cfg.bounded = 1, 2xFP16 engine)");
    cudaStream_t s = h->stream;
    const size_t n = (size_t)d.n;
    if (ub_out && n) CK(h, cudaMemcpyAsync(ub_out, d.ub, n * 4, cudaMemcpyDeviceToDevice, s));
    if (lb_out && n) CK(h, cudaMemcpyAsync(lb_out, d.lb, n * 4, cudaMemcpyDeviceToDevice, s));
    if (p2_out && n) CK(h, cudaMemcpyAsync(p2_out, d.pj2, n * 4, cudaMemcpyDeviceToDevice, s));
    if (Cref_out) CK(h, cudaMemcpyAsync(Cref_out, d.C_ref, (size_t)d.K * d.d * 8, cudaMemcpyDeviceToDevice, s));
    SYNC(h, s);
    return KMEANS_OK;
}

// Two bounded assignments of the current C^t back to back (SPEC.md:126 idempotence):
// the second sees zero drift.  Destructive test hook (overwrites P^{t-1}).
kmeans_status kmeans_bounds_repeat(kmeans_handle* h, float* ub1_out, float* lb1_out, int64_t* scored_out,
                                   int32_t* same_out) {
    LIVE(h);
    const Dev& d = h->d;
    if (!d.ub) FAIL(h, KMEANS_ERR_INVALID, "handle has no bounded engine (cfg.bounded = 1, 2xFP16 engine)");
    if (!scored_out || !same_out) FAIL(h, KMEANS_ERR_INVALID, "NULL output");
    cudaStream_t s = h->stream;
    CK(h, cudaMemcpyAsync(h->st_host, d.st, sizeof(DevState), cudaMemcpyDeviceToHost, s));
    SYNC(h, s);
    if (h->st_host->done || h->st_host->init_mode) FAIL(h, KMEANS_ERR_STATE, "needs a live Algorithm 1 state");
    const int cur = h->st_host->cur;
    long long sc[2];
    for (int k = 0; k < 2; ++k) {
        CK(h, cudaMemsetAsync(h->scratch, 0, h->scratch_bytes, s));
        GEval g{};
        g.branch = 0; g.force = 1; g.prev_mode = 1;
        assign_engine(h, d, g, s);                      // labels -> lab[st->cur], lab_ref = lab[cur ^ 1]
        refine_engine(h, d, g, s);
        CK(h, cudaMemcpyAsync(&sc[k], d.act_count, 8, cudaMemcpyDeviceToHost, s));
        if (k == 0) {
            if (ub1_out && d.n) CK(h, cudaMemcpyAsync(ub1_out, d.ub, (size_t)d.n * 4, cudaMemcpyDeviceToDevice, s));
            if (lb1_out && d.n) CK(h, cudaMemcpyAsync(lb1_out, d.lb, (size_t)d.n * 4, cudaMemcpyDeviceToDevice, s));
            const int nc = cur ^ 1;                     // the bounds now refer to the labels just written
            CK(h, cudaMemcpyAsync(&d.st->cur, &nc, 4, cudaMemcpyHostToDevice, s));
        }
        SYNC(h, s);
    }
    std::vector<int> a(d.n), b(d.n);
    if (d.n) {
        CK(h, cudaMemcpy(a.data(), d.lab[cur], (size_t)d.n * 4, cudaMemcpyDeviceToHost));
        CK(h, cudaMemcpy(b.data(), d.lab[cur ^ 1], (size_t)d.n * 4, cudaMemcpyDeviceToHost));
    }
    const int c0 = cur;
    CK(h, cudaMemcpy(&d.st->cur, &c0, 4, cudaMemcpyHostToDevice));
    scored_out[0] = sc[0]; scored_out[1] = sc[1];
    *same_out = a == b ? 1 : 0;
    return KMEANS_OK;
}

kmeans_status kmeans_update(kmeans_handle* h, const int32_t* labels, const double* C_prev, double* G_out,
                            int64_t* counts_out) {
    Nvtx nvtx_("kmeans_update");
    LIVE(h);
    if ((!labels && h->d.n > 0) || !C_prev || !G_out) FAIL(h, KMEANS_ERR_INVALID, "NULL labels/C_prev/G_out");
    cudaStream_t s = h->stream;
    const Dev& d = h->da;
    CK(h, cudaMemsetAsync(h->scratch, 0, h->scratch_bytes, s));
    CK(h, cudaMemsetAsync(&d.st->label_error, 0, sizeof(int), s));
    GEval g{};
    g.branch = 0; g.force = 1; g.lab_out = const_cast<int*>(labels); g.prev_mode = 1;
    combine(h, d, 2, C_prev, s);                          // max ||c||^2 of C_prev (the energy scale)
    h->launches += launch_update(d, g, s);
    kmeans_status st = allreduce(h, d, 0, s);
    if (st != KMEANS_OK) return st;
    launch_update_G(d, d.packed[0], C_prev, G_out, (long long*)counts_out, s);
    h->launches += 1;
    CK(h, cudaMemcpyAsync(h->done_host, &d.st->label_error, 4, cudaMemcpyDeviceToHost, s));
    SYNC(h, s);
    CK(h, cudaGetLastError());
    if (*h->done_host) FAIL(h, KMEANS_ERR_INVALID, "labels outside [0, K)");
    return KMEANS_OK;
}

kmeans_status kmeans_update_partials(kmeans_handle* h, const int32_t* labels, const int32_t* labels_prev,
                                     const double* C, double* packed_out) {
    LIVE(h);
    if ((!labels && h->d.n > 0) || !C || !packed_out) FAIL(h, KMEANS_ERR_INVALID, "NULL argument");
    cudaStream_t s = h->stream;
    const Dev& d = h->da;
    CK(h, cudaMemsetAsync(h->scratch, 0, h->scratch_bytes, s));
    GEval g{};
    g.branch = 0; g.force = 1; g.lab_out = const_cast<int*>(labels);
    g.prev_mode = labels_prev ? 2 : 1; g.lab_prev = labels_prev;
    combine(h, d, 2, C, s);                               // max ||c||^2 of C (the energy scale)
    h->launches += launch_update(d, g, s);
    h->launches += launch_energy_x(d, g, s);                          // E_local from this rank's sums
    launch_partials_out(d, d.packed[0], packed_out, s);               // unreduced, as doubles
    h->launches += 1;
    SYNC(h, s);
    CK(h, cudaGetLastError());
    return KMEANS_OK;
}

static void fill_info(kmeans_handle* h, kmeans_step_info* info, double* theta) {
    const DevState& S = *h->st_host;
    const TraceRec& r = h->tr_host[0];
    if (info) {
        memset(info, 0, sizeof(*info));
        if (S.trace_len > 0) {
            info->t = r.t; info->m = r.m; info->m_t = r.m_t; info->accepted = r.accepted;
            info->rejected = r.rejected; info->converged = r.converged; info->lloyd = r.lloyd;
            info->energy_cand = r.E_cand; info->energy = r.E_final; info->changed = r.changed;
        } else {   // after line 1
            info->t = 0; info->m = S.m; info->lloyd = 1; info->energy_cand = S.E_cand;
            info->energy = S.E_final;
        }
    }
    if (theta) {
        for (int j = 0; j < h->d.m_max; ++j) theta[j] = j < S.m_t ? S.theta[j] : 0.0;
    }
}

static kmeans_status step_info(kmeans_handle* h, kmeans_step_info* info, double* theta_out) {
    if (info || theta_out) {
        cudaStream_t s = h->stream;
        CK(h, cudaMemcpyAsync(h->st_host, h->d.st, sizeof(DevState), cudaMemcpyDeviceToHost, s));
        SYNC(h, s);
        if (h->st_host->label_error & 2) x_range_error(h);
        if (h->poisoned) return KMEANS_ERR_INVALID;
        const long long n = h->st_host->trace_len;
        if (n > 0)
            CK(h, cudaMemcpy(h->tr_host, h->d.trace + (n - 1), sizeof(TraceRec), cudaMemcpyDeviceToHost));
        fill_info(h, info, theta_out);
    }
    return KMEANS_OK;
}

kmeans_status kmeans_aa_step(kmeans_handle* h, const double* C0, kmeans_step_info* info, double* theta_out) {
    Nvtx nvtx_("kmeans_aa_step");
    LIVE(h);
    kmeans_status st;
    if (C0) st = start(h, C0);
    else st = enqueue_pass(h, h->stream, h->cfg.timing != 0);
    if (st != KMEANS_OK) return st;
    return step_info(h, info, theta_out);
}

// One loop pass with X refreshed from pinned host memory: the H2D copy runs in
// row chunks on a copy stream and the dense tensor-core assignment consumes
// each chunk as it lands, so the transfer overlaps the contraction.
kmeans_status kmeans_aa_step_host(kmeans_handle* h, const float* X_host, int32_t chunks, kmeans_step_info* info,
                                  double* theta_out) {
    Nvtx nvtx_("kmeans_aa_step_host");
    LIVE(h);
    const Dev& d = h->d;
    if (!h->cfg.x_refresh) FAIL(h, KMEANS_ERR_INVALID, "kmeans_aa_step_host needs cfg.x_refresh = 1 at create");
    if (!X_host && d.n > 0) FAIL(h, KMEANS_ERR_INVALID, "X_host is NULL");
    if (chunks < 1) chunks = 1;
    if (chunks > 64) chunks = 64;
    cudaStream_t s = h->stream;
    if (!h->copy_stream) {
        CK(h, cudaStreamCreateWithFlags(&h->copy_stream, cudaStreamNonBlocking));
        CK(h, cudaEventCreateWithFlags(&h->feed_gate, cudaEventDisableTiming));
        CK(h, cudaEventCreateWithFlags(&h->feed_all, cudaEventDisableTiming));
        h->feed_ev.resize(64);
        for (auto& e : h->feed_ev) CK(h, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    const long long T = (d.n + 127) / 128;
    const long long ct = ((T + chunks - 1) / chunks + 1) & ~1LL;      // even: CTA pairs stay inside a chunk
    const int nc = T > 0 ? (int)((T + ct - 1) / ct) : 0;
    CK(h, cudaEventRecord(h->feed_gate, s));                           // earlier work on X is done
    CK(h, cudaStreamWaitEvent(h->copy_stream, h->feed_gate, 0));
    float* X = const_cast<float*>(d.X);
    for (int c = 0; c < nc; ++c) {
        const long long r0 = c * ct * 128, r1 = std::min(d.n, (c + 1) * ct * 128);
        CK(h, cudaMemcpyAsync(X + r0 * d.d, X_host + r0 * d.d, (size_t)(r1 - r0) * d.d * 4, cudaMemcpyHostToDevice,
                              h->copy_stream));
        CK(h, cudaEventRecord(h->feed_ev[c], h->copy_stream));
    }
    // the new rows must stay inside the create-time ranges every scale was derived
    // from (2xFP16 operand scale and tau_abs, fixed-point update and energy scales):
    // one stats pass on the copy stream, checked on the device (label_error bit 2,
    // reported by the next synchronising call)
    CK(h, cudaMemsetAsync(h->xchk, 0, 8, h->copy_stream));
    if (d.x2) CK(h, cudaMemsetAsync(d.x2, 0, 16, h->copy_stream));   // + the new rows' sum ||x_i||^2 (k_energy_x)
    h->launches += launch_xstats_max(d.X, d.n, d.d, h->xchk, h->copy_stream, d.x2, d.x2_e);
    launch_xcheck(d, h->xchk, h->x_stat[0], h->x_stat[1], h->copy_stream);
    h->launches += 1;
    CK(h, cudaEventRecord(h->feed_all, h->copy_stream));
    if (d.ub) CK(h, cudaMemsetAsync(&d.st->bnd_ready, 0, sizeof(int), s));   // new rows: no valid bounds
    CK(h, cudaMemsetAsync(&d.st->sref_valid, 0, sizeof(int), s));            // ... and no valid S(P^{t-1})
    const bool streamed = nc > 0 && !d.ub && (h->path == KMEANS_PATH_TC || h->path == KMEANS_PATH_TC16);
    if (!streamed) {
        CK(h, cudaStreamWaitEvent(s, h->feed_all, 0));
        kmeans_status st = enqueue_pass(h, s, h->cfg.timing != 0);
        if (st != KMEANS_OK) return st;
        return step_info(h, info, theta_out);
    }
    h->feed_chunks = nc;
    h->feed_tiles = ct;
    kmeans_status st = enqueue_pass(h, s, false);
    h->feed_chunks = 0;
    CK(h, cudaStreamWaitEvent(s, h->feed_all, 0));
    if (st != KMEANS_OK) return st;
    return step_info(h, info, theta_out);
}

kmeans_status kmeans_run(kmeans_handle* h, const double* C0, double* C_out, int32_t* labels_out, kmeans_report* rep) {
    Nvtx nvtx_("kmeans_run");
    LIVE(h);
    if (!C0 || !rep) FAIL(h, KMEANS_ERR_INVALID, "C0 or rep is NULL");
    cudaStream_t s = h->stream;
    kmeans_status st = ensure_graph(h);
    if (st != KMEANS_OK) return st;
    CK(h, cudaEventRecord(h->run_ev[0], s));
    st = start(h, C0);
    if (st != KMEANS_OK) return st;
    int batch = 4;
    long long passes = 0;
    while (true) {
        for (int i = 0; i < batch; ++i) {
            CK(h, cudaGraphLaunch(h->pass_exec, s));
            h->launches += h->kernels_per_pass;
        }
        passes += batch;
        CK(h, cudaMemcpyAsync(h->done_host, &h->d.st->done, 4, cudaMemcpyDeviceToHost, s));
        SYNC(h, s);
        if (*h->done_host) break;
        if (passes > (long long)h->cfg.max_iters + 8) FAIL(h, KMEANS_ERR_STATE, "run did not terminate");
        if (batch < 16) batch *= 2;
    }
    CK(h, cudaEventRecord(h->run_ev[1], s));
    if (C_out) CK(h, cudaMemcpyAsync(C_out, h->d.C, (size_t)h->d.K * h->d.d * 8, cudaMemcpyDeviceToDevice, s));
    CK(h, cudaMemcpyAsync(h->st_host, h->d.st, sizeof(DevState), cudaMemcpyDeviceToHost, s));
    SYNC(h, s);
    const DevState& S = *h->st_host;
    // the conditional branch-B body ran only on the passes that rejected an iterate
    h->launches -= (passes - std::min<long long>(passes, S.n_rejected)) * h->kernels_b;
    if (S.label_error & 2) { x_range_error(h); return KMEANS_ERR_INVALID; }
    if (labels_out && h->d.n > 0)
        CK(h, cudaMemcpyAsync(labels_out, h->d.lab[S.cur], (size_t)h->d.n * 4, cudaMemcpyDeviceToDevice, s));
    float ms = 0.f;
    CK(h, cudaEventElapsedTime(&ms, h->run_ev[0], h->run_ev[1]));
    SYNC(h, s);
    memset(rep, 0, sizeof(*rep));
    rep->converged = S.converged;
    rep->iters = S.converged ? S.t + 1 : S.t;
    rep->n_rejected = S.n_rejected;
    rep->n_accepted = S.n_accepted;
    rep->n_assign = S.n_assign;
    rep->m_final = S.m;
    rep->energy = S.E_final;
    rep->mse = S.E_final / (double)h->n_global;
    rep->seconds = ms / 1e3;
    return KMEANS_OK;
}

kmeans_status kmeans_get_centroids(kmeans_handle* h, double* C_out, int32_t* labels_out) {
    LIVE(h);
    cudaStream_t s = h->stream;
    if (C_out) CK(h, cudaMemcpyAsync(C_out, h->d.C, (size_t)h->d.K * h->d.d * 8, cudaMemcpyDeviceToDevice, s));
    if (labels_out) {
        CK(h, cudaMemcpyAsync(h->st_host, h->d.st, sizeof(DevState), cudaMemcpyDeviceToHost, s));
        SYNC(h, s);
        // after a pass the last assignment is P^t = lab[cur ^ 1] unless the run stopped (done)
        const DevState& S = *h->st_host;
        int which = S.done ? S.cur : (S.cur ^ 1);
        CK(h, cudaMemcpyAsync(labels_out, h->d.lab[which], (size_t)h->d.n * 4, cudaMemcpyDeviceToDevice, s));
    }
    return KMEANS_OK;
}

kmeans_status kmeans_state_export(kmeans_handle* h, kmeans_state* out) {
    LIVE(h);
    if (!out) FAIL(h, KMEANS_ERR_INVALID, "NULL state");
    cudaStream_t s = h->stream;
    CK(h, cudaMemcpyAsync(h->st_host, h->d.st, sizeof(DevState), cudaMemcpyDeviceToHost, s));
    SYNC(h, s);
    const DevState& S = *h->st_host;
    const Dev& d = h->d;
    const size_t KD = (size_t)d.K * d.d;
    out->hist_count = S.hist_count; out->m = S.m; out->lloyd = S.lloyd; out->done = S.done; out->t = S.t;
    out->E1 = S.E1; out->E2 = S.E2;
    out->n_accepted = S.n_accepted; out->n_rejected = S.n_rejected; out->n_assign = S.n_assign;
    if (out->C) CK(h, cudaMemcpy(out->C, d.C, KD * 8, cudaMemcpyDeviceToHost));
    // between passes the newest history entry is (G^{t-1}, F^{t-1})
    for (int j = 0; j < S.hist_count; ++j) {
        const long long slot = ((S.t - 1 - j) % d.H + d.H) % d.H;
        if (out->Ghist) CK(h, cudaMemcpy(out->Ghist + j * KD, d.Gring + slot * KD, KD * 8, cudaMemcpyDeviceToHost));
        if (out->Fhist) CK(h, cudaMemcpy(out->Fhist + j * KD, d.Fring + slot * KD, KD * 8, cudaMemcpyDeviceToHost));
    }
    if (out->fallback && S.hist_count > 0) {
        const long long slot = ((S.t - 1) % d.H + d.H) % d.H;
        CK(h, cudaMemcpy(out->fallback, d.Gring + slot * KD, KD * 8, cudaMemcpyDeviceToHost));
    }
    if (out->labels_prev && d.n > 0) {
        // between passes P^{t-1} = lab[cur ^ 1]; a finished run (converged or max_iters)
        // did not flip cur, so its final P^t is lab[cur] (kmeans_get_centroids agrees)
        const int which = S.done ? S.cur : (S.cur ^ 1);
        CK(h, cudaMemcpy(out->labels_prev, d.lab[which], (size_t)d.n * 4, cudaMemcpyDeviceToHost));
    }
    if (out->gram)
        for (int a = 0; a < d.H; ++a)
            for (int b = 0; b < d.H; ++b) out->gram[a * d.H + b] = S.gram[a * d.H + b];
    return KMEANS_OK;
}

kmeans_status kmeans_state_import(kmeans_handle* h, const kmeans_state* st) {
    LIVE(h);
    const Dev& d = h->d;
    if (!st || !st->C || (st->hist_count > 0 && (!st->Ghist || !st->Fhist)) || (d.n > 0 && !st->labels_prev))
        FAIL(h, KMEANS_ERR_INVALID, "NULL state buffer");
    if (st->hist_count < 0 || st->hist_count > d.H) FAIL(h, KMEANS_ERR_INVALID, "hist_count outside [0, m_max + 1]");
    if (st->m < 0 || st->m > d.m_max) FAIL(h, KMEANS_ERR_INVALID, "m outside [0, m_max]");
    if (st->t < 1) FAIL(h, KMEANS_ERR_INVALID, "t < 1 (export after Algorithm 1 line 1)");
    cudaStream_t s = h->stream;
    const size_t KD = (size_t)d.K * d.d;
    SYNC(h, s);
    // history into the ring slots it came from: entry j = (G^{t-1-j}, F^{t-1-j})
    for (int j = 0; j < st->hist_count; ++j) {
        const long long slot = ((st->t - 1 - j) % d.H + d.H) % d.H;
        CK(h, cudaMemcpy(d.Gring + slot * KD, st->Ghist + j * KD, KD * 8, cudaMemcpyHostToDevice));
        CK(h, cudaMemcpy(d.Fring + slot * KD, st->Fhist + j * KD, KD * 8, cudaMemcpyHostToDevice));
    }
    CK(h, cudaMemcpy(d.C, st->C, KD * 8, cudaMemcpyHostToDevice));
    // cur = 0 below: a live state's P^{t-1} goes to lab[cur ^ 1]; a finished one's
    // final labels to lab[cur] (the buffers export and get_centroids read)
    if (d.n > 0) CK(h, cudaMemcpy(d.lab[st->done ? 0 : 1], st->labels_prev, (size_t)d.n * 4, cudaMemcpyHostToDevice));
    // the control state, on top of the current device state (keeps engine-side fields)
    CK(h, cudaMemcpy(h->st_host, d.st, sizeof(DevState), cudaMemcpyDeviceToHost));
    DevState S = *h->st_host;
    S.t = st->t; S.m = st->m; S.lloyd = st->lloyd; S.E1 = st->E1; S.E2 = st->E2;
    S.E_final = st->E1; S.E_cand = st->E1;
    S.done = st->done; S.converged = 0; S.cur = 0; S.init_mode = 0; S.reject = 0;
    S.hist_count = st->hist_count; S.n_accepted = st->n_accepted; S.n_rejected = st->n_rejected;
    S.n_assign = st->n_assign; S.trace_len = 0; S.final_traced = 0; S.label_error = 0;
    S.bnd_ready = 0; S.bnd_use = 0; S.rows_scored = 0; S.rows_total = 0;
    S.sref_valid = 0; S.use_delta = 0;                                // no S(P^{t-1}) for the imported labels
    if (st->gram) {
        for (int a = 0; a < d.H; ++a)
            for (int b = 0; b < d.H; ++b) S.gram[a * d.H + b] = st->gram[a * d.H + b];
    } else {
        // recompute <dF(a), dF(b)> for the window from the host history (fp64)
        const int W = st->hist_count - 1;                         // differences available
        for (int a = 0; a < W; ++a)
            for (int b = 0; b <= a; ++b) {
                double v = 0.0;
                for (size_t e = 0; e < KD; ++e) {
                    const double da = st->Fhist[a * KD + e] - st->Fhist[(a + 1) * KD + e];
                    const double db = st->Fhist[b * KD + e] - st->Fhist[(b + 1) * KD + e];
                    v += da * db;
                }
                const long long sa = ((st->t - 1 - a) % d.H + d.H) % d.H, sb = ((st->t - 1 - b) % d.H + d.H) % d.H;
                S.gram[sa * d.H + sb] = v;
                S.gram[sb * d.H + sa] = v;
            }
    }
    CK(h, cudaMemcpy(d.st, &S, sizeof(DevState), cudaMemcpyHostToDevice));
    combine(h, d, 2, d.C, s);                                     // operand prep of C^t
    SYNC(h, s);
    CK(h, cudaGetLastError());
    return KMEANS_OK;
}

kmeans_status kmeans_debug_check_canaries(kmeans_handle* h, int64_t* bad_bytes, int64_t* n_guards) {
    LIVE(h);
    if (!bad_bytes) FAIL(h, KMEANS_ERR_INVALID, "NULL output");
    SYNC(h, h->stream);
    std::vector<unsigned char> buf(256);
    long long bad = 0;
    for (size_t g : h->guards) {
        CK(h, cudaMemcpy(buf.data(), h->ws_base + g, 256, cudaMemcpyDeviceToHost));
        for (unsigned char c : buf) bad += c != CANARY;
    }
    *bad_bytes = bad;
    if (n_guards) *n_guards = (int64_t)h->guards.size();
    return KMEANS_OK;
}

kmeans_status kmeans_trace_export(kmeans_handle* h, kmeans_step_info* out, int64_t cap, int64_t* n_out) {
    LIVE(h);
    if (!n_out || (cap > 0 && !out)) FAIL(h, KMEANS_ERR_INVALID, "NULL output");
    cudaStream_t s = h->stream;
    CK(h, cudaMemcpyAsync(h->st_host, h->d.st, sizeof(DevState), cudaMemcpyDeviceToHost, s));
    SYNC(h, s);
    const long long n = h->st_host->trace_len;
    *n_out = n;
    const long long m = std::min<long long>(n, cap);
    if (m <= 0) return KMEANS_OK;
    std::vector<TraceRec> tr((size_t)m);
    CK(h, cudaMemcpy(tr.data(), h->d.trace, (size_t)m * sizeof(TraceRec), cudaMemcpyDeviceToHost));
    for (long long i = 0; i < m; ++i) {
        const TraceRec& r = tr[(size_t)i];
        kmeans_step_info& o = out[i];
        memset(&o, 0, sizeof(o));
        o.t = r.t; o.m = r.m; o.m_t = r.m_t; o.accepted = r.accepted; o.rejected = r.rejected;
        o.converged = r.converged; o.lloyd = r.lloyd; o.energy_cand = r.E_cand; o.energy = r.E_final;
        o.changed = r.changed;
    }
    return KMEANS_OK;
}

kmeans_status kmeans_assign_timing(kmeans_handle* h, double* ms_total, int64_t* launches) {
    LIVE(h);
    SYNC(h, h->stream);
    double tot = 0.0;
    for (size_t i = 0; i < h->ev_used; ++i) {
        float ms = 0.f;
        CK(h, cudaEventElapsedTime(&ms, h->ev[i].first, h->ev[i].second));
        tot += ms;
    }
    if (ms_total) *ms_total = tot;
    if (launches) *launches = (int64_t)h->ev_used;
    h->ev_used = 0;
    return KMEANS_OK;
}

kmeans_status kmeans_update_timing(kmeans_handle* h, double* ms_total, int64_t* launches) {
    LIVE(h);
    SYNC(h, h->stream);
    double tot = 0.0;
    for (size_t i = 0; i < h->uev_used; ++i) {
        float ms = 0.f;
        CK(h, cudaEventElapsedTime(&ms, h->uev[i].first, h->uev[i].second));
        tot += ms;
    }
    if (ms_total) *ms_total = tot;
    if (launches) *launches = (int64_t)h->uev_used;
    h->uev_used = 0;
    return KMEANS_OK;
}

int64_t kmeans_launch_count(const kmeans_handle* h) { return h ? h->launches : 0; }

// K-Means++ seeding (seed.cu, reading R-A27): K rounds, each one pass over X
// plus three small kernels; with nranks > 1 three tiny allreduces per round
// (max D2, the ranks' weight totals, the chosen row).
kmeans_status kmeans_seed_pp(kmeans_handle* h, const double* u, float* C_out, int64_t* idx_out) {
    Nvtx nvtx_("kmeans_seed_pp");
    LIVE(h);
    const Dev& d = h->d;
    const int K = d.K;
    if (!u || !C_out) FAIL(h, KMEANS_ERR_INVALID, "NULL u or C_out");
    for (int r = 0; r < K; ++r)
        if (!(u[r] >= 0.0 && u[r] < 1.0)) FAIL(h, KMEANS_ERR_INVALID, "u outside [0, 1)");
    cudaStream_t s = h->stream;
    const long long N = h->n_global;
    long long offset = 0;                               // this rank's first global row
    if (h->comm) {
        std::vector<long long> nl(h->nranks, 0);
        nl[h->rank] = d.n;
        CK(h, cudaMemcpyAsync(d.seed_T, nl.data(), 8 * h->nranks, cudaMemcpyHostToDevice, s));
        NK(h, ncclAllReduce(d.seed_T, d.seed_T, h->nranks, ncclInt64, ncclSum, h->comm, s));
        CK(h, cudaMemcpyAsync(nl.data(), d.seed_T, 8 * h->nranks, cudaMemcpyDeviceToHost, s));
        SYNC(h, s);
        for (int q = 0; q < h->rank; ++q) offset += nl[q];
    }
    CK(h, cudaMemcpyAsync(d.seed_u, u, 8 * (size_t)K, cudaMemcpyHostToDevice, s));
    CK(h, cudaMemsetAsync(&d.st->seed_max, 0, 16, s));   // seed_max, seed_err
    const double a = h->x_gamax;
    int e = 0;
    if (a > 0.0) frexp(4.0 * a * a, &e);                 // (2 max|x|)^2 < 2^e
    const double scale = ldexp(1.0, 50 - e);
    int log2n = 0;
    while ((1LL << log2n) < N) ++log2n;
    long long i0 = (long long)floor(u[0] * (double)N);
    if (i0 > N - 1) i0 = N - 1;
    const long long loc = (i0 >= offset && i0 < offset + d.n) ? i0 - offset : -1;
    launch_seed_first(d, loc, i0, s);
    if (h->comm) NK(h, ncclAllReduce(d.seed_x, d.seed_x, d.d + 2, ncclInt32, ncclSum, h->comm, s));
    launch_seed_commit(d, C_out, 0, s);
    h->launches += 2;
    for (int r = 1; r < K; ++r) {
        h->launches += launch_seed_dist(d, C_out, r - 1, scale, s) - 1;   // D2 against the newest center r - 1
        if (h->comm)
            NK(h, ncclAllReduce(&d.st->seed_max, &d.st->seed_max, 1, ncclInt64, ncclMax, h->comm, s));
        launch_seed_weights(d, log2n, h->rank, h->nranks, s);
        if (h->comm) NK(h, ncclAllReduce(d.seed_T, d.seed_T, h->nranks, ncclInt64, ncclSum, h->comm, s));
        launch_seed_select(d, r, log2n, h->rank, h->nranks, offset, s);
        if (h->comm) NK(h, ncclAllReduce(d.seed_x, d.seed_x, d.d + 2, ncclInt32, ncclSum, h->comm, s));
        launch_seed_commit(d, C_out, r, s);
        h->launches += 5;
        if ((r & 255) == 0) CK(h, cudaGetLastError());
    }
    int err = 0;
    CK(h, cudaMemcpyAsync(&err, &d.st->seed_err, 4, cudaMemcpyDeviceToHost, s));
    if (idx_out) CK(h, cudaMemcpyAsync(idx_out, d.seed_idx, 8 * (size_t)K, cudaMemcpyDeviceToHost, s));
    SYNC(h, s);
    CK(h, cudaGetLastError());
    if (err) FAIL(h, KMEANS_ERR_INVALID, "fewer distinct samples than K (every remaining D^2 is 0)");
    return KMEANS_OK;
}

kmeans_status kmeans_bounded_stats(kmeans_handle* h, int64_t* rows_scored, int64_t* rows_total) {
    LIVE(h);
    if (!rows_scored || !rows_total) FAIL(h, KMEANS_ERR_INVALID, "NULL output");
    CK(h, cudaMemcpyAsync(h->st_host, h->d.st, sizeof(DevState), cudaMemcpyDeviceToHost, h->stream));
    SYNC(h, h->stream);
    *rows_scored = h->st_host->rows_scored;
    *rows_total = h->st_host->rows_total;
    return KMEANS_OK;
}

kmeans_status kmeans_update_stats(kmeans_handle* h, int64_t* n_evals, int64_t* n_incremental, int64_t* rows_moved) {
    LIVE(h);
    if (!n_evals || !n_incremental || !rows_moved) FAIL(h, KMEANS_ERR_INVALID, "NULL output");
    CK(h, cudaMemcpyAsync(h->st_host, h->d.st, sizeof(DevState), cudaMemcpyDeviceToHost, h->stream));
    SYNC(h, h->stream);
    *n_evals = h->d.sref ? h->st_host->n_upd : 0;
    *n_incremental = h->d.sref ? h->st_host->n_delta : 0;
    *rows_moved = h->d.sref ? h->st_host->rows_moved : 0;
    return KMEANS_OK;
}

kmeans_status kmeans_last_flagged(kmeans_handle* h, int64_t* flagged) {
    LIVE(h);
    if (!flagged) return KMEANS_ERR_INVALID;
    long long v[2], pr[2];
    SYNC(h, h->stream);
    CK(h, cudaMemcpy(v, h->d.flag_count, 16, cudaMemcpyDeviceToHost));
    CK(h, cudaMemcpy(pr, h->d.pair_count, 16, cudaMemcpyDeviceToHost));
    *flagged = v[0] + pr[0];                            // candidate-pass rows + two-centroid rows
    return KMEANS_OK;
}

kmeans_status kmeans_comm_info(kmeans_handle* h, int32_t* mode, int32_t* lsa_size) {
    LIVE(h);
    if (!mode) FAIL(h, KMEANS_ERR_INVALID, "NULL mode");
    *mode = h->fused ? fused_mode(h->fused) : (h->comm ? 0 : -1);
    if (lsa_size) *lsa_size = h->fused ? fused_lsa_size(h->fused) : 0;
    return KMEANS_OK;
}

const char* kmeans_assign_path_name(const kmeans_handle* h) {
    if (!h) return "none";
    return h->path == KMEANS_PATH_TC ? "tc" : h->path == KMEANS_PATH_TC16 ? "tc16" : "simt";
}

kmeans_status kmeans_destroy(kmeans_handle* h) {
    Nvtx nvtx_("kmeans_destroy");
    if (!h) return KMEANS_ERR_INVALID;
    if (g_prof) prof_dump();
    if (h->d.dbg_ts) {                                                 // AAKM_TC_TRACE: dump the stamps
        std::vector<unsigned long long> ts(2 * 8 * 256);
        cudaDeviceSynchronize();
        cudaMemcpy(ts.data(), h->d.dbg_ts, ts.size() * 8, cudaMemcpyDeviceToHost);
        if (FILE* f = fopen(getenv("AAKM_TC_TRACE"), "w")) {
            for (int b = 0; b < 2; ++b)
                for (int it = 0; it < 256; ++it) {
                    fprintf(f, "%d %d", b, it);
                    for (int e = 0; e < 8; ++e) fprintf(f, " %llu", ts[(b * 8 + e) * 256 + it]);
                    fprintf(f, "\n");
                }
            fclose(f);
        }
        if (const char* sp = getenv("AAKM_SOLVE_TRACE")) {            // k_solve phase clocks (probe builds)
            std::vector<unsigned long long> sv(256);
            cudaMemcpy(sv.data(), h->d.dbg_ts + 2 * 8 * 256, 256 * 8, cudaMemcpyDeviceToHost);
            if (FILE* f = fopen(sp, "w")) {
                for (int i = 0; i < 256; ++i) fprintf(f, "%llu\n", sv[i]);
                fclose(f);
            }
        }
        cudaFree(h->d.dbg_ts);
    }
    release(h, !h->poisoned);
    return KMEANS_OK;
}

const char* kmeans_last_error(const kmeans_handle* h) {
    if (!h) return g_create_err.c_str();
    return h->err.c_str();
}

}  // extern "C"
