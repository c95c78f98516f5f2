/*
 * aakm.h -- C ABI of the B200-native Anderson-accelerated Lloyd K-Means hot
 * path (arXiv 1805.10638).  Library: paper_1805_10638_b200/libaakm.so
 * (hand-written sm_100a CUDA + NCCL; no torch types, no CPU fallback).
 *
 * Notation follows the paper: samples X = {x_i} (N x d), centroids
 * C = [c_1..c_K] (K x d), assignment P = {rho_i}, energy E (Eq. 1,
 * PAPER.md:14), Lloyd map G = Update o Assign (Eq. 6), residual
 * F = G - C, Anderson window m, Algorithm 1
 * (PAPER.md:107-160).  Readings of ambiguous passages are DESIGN.md R-A*.
 *
 * Conventions for every entry point:
 *  - Array pointers are DEVICE pointers unless marked (host).
 *  - Row-major layouts: X is n_local x d float32 (the samples, BASELINE.json's
 *    fp32 data); centroids C, G, C0 are K x d float64 (centroid-major): the
 *    whole Algorithm 1 state -- C^t, the fallback, the G/F history -- is fp64
 *    on the device (DESIGN.md R-A17); labels are int32 in [0, K).
 *  - Ownership: X and the workspace are BORROWED from the caller and must stay
 *    alive and unmodified until kmeans_destroy (the one exception is opt-in:
 *    with cfg.x_refresh = 1, kmeans_aa_step_host rewrites X from the caller's
 *    host copy).  The library allocates no
 *    device memory of its own except NCCL's internal buffers (nranks > 1).
 *    Outputs go to caller buffers.
 *  - Streams: all work is enqueued on the stream given to kmeans_create.
 *    Calls returning host scalars synchronise that stream before returning;
 *    the others are asynchronous.  One host thread at a time per handle.
 *  - SPMD: with nranks > 1, assign/update/aa_step/run are COLLECTIVE (like
 *    NCCL calls): every rank calls them in the same order; X is the rank's
 *    contiguous row shard; C and config are identical on all ranks.  Ranks
 *    combine [S | N | E | changed] (exact int64 fixed point) with one
 *    ncclAllReduce per G-evaluation;
 *    the Anderson step is replicated (deterministic kernels, identical bytes).
 *  - Errors: KMEANS_ERR_INVALID is returned before any work is enqueued (null
 *    required pointer, d < 1, k < 1, k > n_global, m0 < 0, m0 > m_max,
 *    m_max > KMEANS_M_MAX, eps1 < 0 or eps1 >= eps2, workspace too small,
 *    bad rank/nranks).  CUDA or NCCL failures return ERR_CUDA / ERR_NCCL and
 *    poison the handle: afterwards only kmeans_destroy is valid, everything
 *    else returns KMEANS_ERR_STATE.  Reaching max_iters is not an error
 *    (report.converged = 0).  kmeans_last_error() gives the message.
 */
#ifndef AAKM_H
#define AAKM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(AAKM_BUILD)
#define AAKM_API __attribute__((visibility("default")))
#else
#define AAKM_API
#endif

#define KMEANS_M_MAX 30          /* m_bar of PAPER.md:177; ring = m_max + 1 slots */
#define KMEANS_ABI_VERSION 4

typedef struct kmeans_handle kmeans_handle;
typedef struct CUstream_st *kmeans_stream_t;   /* == cudaStream_t */

typedef enum {
    KMEANS_OK = 0,
    KMEANS_ERR_INVALID = 1,
    KMEANS_ERR_CUDA = 2,
    KMEANS_ERR_NCCL = 3,
    KMEANS_ERR_NOMEM = 4,
    KMEANS_ERR_STATE = 5
} kmeans_status;

/* Assignment engine selection (kmeans_config.assign_path). */
enum {
    KMEANS_PATH_AUTO = 0,   /* tcgen05 2xFP16 for d in {64,128}, 3xTF32 for other d % 32 == 0 <= 128, else SIMT */
    KMEANS_PATH_SIMT = 1,   /* register-tiled FP32 FFMA kernel                          */
    KMEANS_PATH_TC = 2,     /* tcgen05/TMEM 3xTF32 tile GEMM (requires d % 32 == 0, d <= 128) */
    KMEANS_PATH_TC16 = 3    /* tcgen05/TMEM 2xFP16 split (power-of-two scaled), d in {64, 128} */
};

/* Algorithm 1 settings.  Defaults (kmeans_config_default): PAPER.md:177
 * (eps1 = 0.02, eps2 = 0.5, m_max = 30, m0 = 2), dynamic m on. */
typedef struct {
    int32_t m0;          /* initial m                         */
    int32_t m_max;       /* m_bar, <= KMEANS_M_MAX                               */
    double eps1;         /* ratio below which m decreases     */
    double eps2;         /* ratio above which m increases     */
    int32_t dynamic_m;   /* 1 = Algorithm 1; 0 = fixed m            */
    int32_t max_iters;   /* cap on passes t (not an error when reached)           */
    double ridge;        /* lambda on the unit-diagonal scaled Gram (R-A14)       */
    int32_t assign_path; /* KMEANS_PATH_*                                        */
    int32_t timing;      /* 1 = CUDA events around each assignment and update   */
    int32_t bounded;     /* 1 = Hamerly-bounded assignment in the Algorithm 1
                            passes (aa_step / run; 2xFP16 engine only, otherwise
                            ignored): per row an upper bound on the distance to
                            its centroid and a lower bound on every other one,
                            moved by the centroid shifts (the paper's Assignment-
                            Step is Hamerly-pruned); rows the
                            bounds prove unchanged keep their label, the rest run
                            through the tensor engine as a gathered row list.
                            Labels stay exact.  Default 0 (dense: bench.py's
                            dist-evals/s metric counts N*K per pass).            */
    int32_t x_refresh;   /* 1 = X is a staging buffer that kmeans_aa_step_host
                            may overwrite from host memory (the e2e path); the
                            new rows must stay inside the create-time ranges
                            (max |x_ik|, max ||x_i||), which a device check
                            enforces.  0 (default): X is never written, and
                            kmeans_aa_step_host returns INVALID.                 */
    int32_t comm_always; /* 1 = build an NCCL communicator even when nranks == 1
                            (a real 1-rank communicator: every allreduce of the
                            data plane, graph-captured ones included, runs
                            through NCCL; results are bitwise those of the
                            communicator-free path).  With a communicator, every
                            synchronising call polls ncclCommGetAsyncError and
                            aborts after AAKM_COMM_TIMEOUT_S seconds (default
                            600) instead of blocking on a failed peer.           */
    int32_t fused_comm;  /* 1 = f4: the per-G-evaluation combine fused into the
                            update's flushes (NCCL 2.28 device API): the packed
                            [S|N|E|changed] vectors live in an NCCL symmetric
                            window and every flush adds into ALL ranks' replicas
                            (multimem.red through the NVLS multicast address, or
                            system-scope reds to each LSA peer), fenced by two
                            device barriers per G-evaluation -- no allreduce
                            launch.  Needs a communicator (nranks > 1 or
                            comm_always) whose ranks share one NVLink domain.
                            Same bytes as the allreduce path.                    */
} kmeans_config;

/* Result of kmeans_run (fields per DESIGN.md R-A19). */
typedef struct {
    int64_t iters;       /* t_final + 1 = main-sequence G evaluations             */
    int64_t n_assign;    /* assignment passes = iters + n_rejected                */
    int64_t n_accepted;  /* accelerated iterates accepted by the guard            */
    int64_t n_rejected;  /* accelerated iterates rejected      */
    int32_t converged;   /* 1 = partition repeated (rule R3); 0 = max_iters       */
    int32_t m_final;
    double energy;       /* E(P, C) of the returned C (Eq. 1), global            */
    double mse;          /* energy / n_global (R-A20)                            */
    double seconds;      /* device time of the run (CUDA events)                 */
} kmeans_report;

/* One loop pass of Algorithm 1 (kmeans_aa_step). */
typedef struct {
    int64_t t;           /* pass index that was executed                          */
    int32_t m;           /* m after the dynamic adjustment                        */
    int32_t m_t;         /* min(m, t) columns used                 */
    int32_t accepted;    /* accelerated iterate accepted this pass                */
    int32_t rejected;    /* accelerated iterate rejected -> Lloyd fallback        */
    int32_t converged;   /* partition repeated: C is a fixed point of G           */
    int32_t lloyd;       /* next iterate C^{t+1} is a plain Lloyd iterate         */
    double energy_cand;  /* E(C^t) of the candidate (pre-guard)                   */
    double energy;       /* E^t after the guard                    */
    int64_t changed;     /* #{i : rho_i^t != rho_i^{t-1}} of the final P^t         */
} kmeans_step_info;

/* Algorithm 1 state, for checkpoint/resume and lockstep parity tests.
 * All pointers are HOST buffers supplied by the caller (fp64, the device
 * state verbatim):
 *   C, fallback: K*d; Ghist, Fhist: (m_max+1)*K*d, entry 0 = newest
 *   (G^t, F^t), entry j = (G^{t-j}, F^{t-j}); labels_prev: n_local. */
typedef struct {
    double *C;           /* C^t, the iterate the next pass evaluates              */
    double *fallback;    /* C_AU^t = G^{t-1} (R-A3)                               */
    double *Ghist;
    double *Fhist;
    int32_t *labels_prev;/* P^{t-1}; for a finished state (done) the final P^t    */
    int32_t hist_count;  /* valid history entries                                 */
    int32_t m;
    int32_t lloyd;       /* C^t is a Lloyd iterate (theta == 0)                   */
    int32_t done;        /* converged or max_iters reached                        */
    int64_t t;
    double E1, E2;       /* E^{t-1}, E^{t-2} (post-guard)                         */
    int64_t n_accepted, n_rejected, n_assign;
    double *gram;        /* (m_max+1)^2 doubles, nullable: the cached Gram entries
                            <dF(a), dF(b)> indexed by ring slot (a mod (m_max+1));
                            opaque -- export fills it, import restores it so a
                            resumed run repeats the uninterrupted one; NULL on
                            import recomputes it from Fhist on the host          */
} kmeans_state;

/* Fill cfg with the defaults above.  Errors: INVALID if cfg is NULL. */
AAKM_API kmeans_status kmeans_config_default(kmeans_config *cfg /*host*/);

/* Bytes of device workspace kmeans_create needs for this shard.
 * Errors: INVALID on bad sizes/config or NULL bytes. */
AAKM_API kmeans_status kmeans_workspace_size(int64_t n_local, int32_t d, int32_t k,
                                    const kmeans_config *cfg /*host*/, size_t *bytes /*host*/);

/* 128-byte NCCL unique id (call on rank 0, broadcast to the other ranks). */
AAKM_API kmeans_status kmeans_nccl_unique_id(void *uid128 /*host, 128 B*/);

/* Create a handle over this rank's shard X (n_local x d, device, borrowed).
 * n_global = sum of n_local over ranks.  workspace: >= kmeans_workspace_size
 * bytes of device memory, 256-B aligned, borrowed.  uid128 must be NULL iff
 * nranks == 1.  Collective when nranks > 1 (NCCL communicator init). */
AAKM_API kmeans_status kmeans_create(kmeans_handle **out /*host*/, const float *X, int64_t n_local,
                            int64_t n_global, int32_t d, int32_t k,
                            const kmeans_config *cfg /*host*/, void *workspace,
                            size_t workspace_bytes, int32_t rank, int32_t nranks,
                            const void *uid128 /*host or NULL*/, kmeans_stream_t stream);

/* Assignment step, Eq. (3), plus the energy E(P, C) (Eq. 1)
 * and the number of labels that differ from labels_prev.
 * C: K x d.  labels_out: n_local (exact nearest centroid, lowest index on
 * exact fp64 ties).  energy_out / changed_out are GLOBAL (allreduced) host
 * scalars, may be NULL; changed is 0 when labels_prev is NULL.  Synchronises. */
AAKM_API kmeans_status kmeans_assign(kmeans_handle *h, const double *C, const int32_t *labels_prev,
                            int32_t *labels_out, double *energy_out /*host*/,
                            int64_t *changed_out /*host*/);

/* Update step, Eq. (4): G_j = mean of {x_i : rho_i = j} over
 * all ranks; an empty cluster keeps C_prev's row (R-A15).  labels: n_local in
 * [0, K) (out-of-range -> INVALID after the sync).  counts_out: K int64
 * device, nullable.  Synchronises (to report label errors). */
AAKM_API kmeans_status kmeans_update(kmeans_handle *h, const int32_t *labels, const double *C_prev,
                            double *G_out, int64_t *counts_out);

/* Algorithm 1, one step.  C0 != NULL: line 1 -- P^0 =
 * Assign(C^0), C^1 = G(C^0), F^0 = C^1 - C^0, E^0 = +inf, m = m0, t = 1.
 * C0 == NULL: one loop pass t under rule R3 (R-A10).
 * info/theta_out (host, nullable; theta_out >= m_max doubles): when either is
 * non-NULL the call synchronises; otherwise it is asynchronous. */
AAKM_API kmeans_status kmeans_aa_step(kmeans_handle *h, const double *C0, kmeans_step_info *info /*host*/,
                             double *theta_out /*host*/);

/* Algorithm 1 to convergence (rule R3) or max_iters, without a host sync per
 * pass (CUDA-graph replay, device-side control).  C_out: K x d (global,
 * identical on all ranks), labels_out: n_local; both nullable.  Synchronises. */
AAKM_API kmeans_status kmeans_run(kmeans_handle *h, const double *C0, double *C_out, int32_t *labels_out,
                         kmeans_report *rep /*host*/);

/* Current iterate C^t and the labels of the last assignment (device copies).
 * Asynchronous. */
AAKM_API kmeans_status kmeans_get_centroids(kmeans_handle *h, double *C_out, int32_t *labels_out);

/* Checkpoint / lockstep hooks (host buffers, see kmeans_state).  Synchronise.
 * export: the state between two passes (after kmeans_aa_step / kmeans_run).
 * import: replaces the Algorithm 1 state of this handle (same X, K, d and
 * m_max as the exporter; nranks > 1: every rank imports its own export); the
 * next kmeans_aa_step(NULL) continues pass t.  Errors: INVALID for NULL C /
 * fallback / history buffers, hist_count outside [0, m_max + 1], m outside
 * [0, m_max], t < 1. */
AAKM_API kmeans_status kmeans_state_export(kmeans_handle *h, kmeans_state *st /*host*/);
AAKM_API kmeans_status kmeans_state_import(kmeans_handle *h, const kmeans_state *st /*host*/);

/* Test hook for the data-parallel partition logic: this rank's UNREDUCED
 * partials [S (K*d, S_j = sum of x_i over rho_i = j) | N (K) | E_local |
 * changed] as K*d + K + 2 doubles (device): S from the exact fixed-point sums,
 * E_local = sum over this rank's rows of ||x_i - c_{rho_i}||^2 (so the ranks'
 * values sum to the global E; label-sorted engine, n_global >= 65536: through
 * sum ||x_i||^2 + sum_j (N_j ||c_j||^2 - 2 c_j . S_j) of this rank's sums,
 * DESIGN.md R-A30).  labels_prev nullable (changed = 0).
 * Synchronises. */
AAKM_API kmeans_status kmeans_update_partials(kmeans_handle *h, const int32_t *labels,
                                     const int32_t *labels_prev, const double *C,
                                     double *packed_out);

/* K-Means++ seeding (Arthur & Vassilvitskii 2007, which the paper uses among
 * its seeders: PAPER.md:44,347) of the handle's K centers.
 *   u       host, K uniforms in [0, 1) (the caller's random numbers): center 0
 *           is global sample floor(u[0] N); center r >= 1 is drawn by inverse
 *           CDF with u[r] from weights w_i proportional to D(x_i)^2, the squared
 *           distance to the nearest chosen center, in the fixed point of
 *           DESIGN.md reading R-A27 (so every rank count draws the same
 *           samples, and samples with D = 0 are never drawn).
 *   C_out   device, K x d fp32 row-major, caller-owned: the chosen samples.
 *   idx_out host, K int64 (nullable): their global row indices.
 * Collective when nranks > 1 (three small allreduces per center). Uses the
 * handle's X and workspace; does not touch the Algorithm 1 state.  Rows whose
 * D^2 provably cannot drop (triangle inequality over the chosen centers) are
 * not re-read; the weights are the same integers (AAKM_SEED_PRUNE=0: every row).
 * Synchronises. Errors: INVALID for NULL u / C_out, a u outside [0, 1), or
 * fewer than K distinct samples (every remaining D^2 = 0). */
AAKM_API kmeans_status kmeans_seed_pp(kmeans_handle *h, const double *u /*host*/, float *C_out,
                                      int64_t *idx_out /*host*/);

/* One loop pass of Algorithm 1 (as kmeans_aa_step(h, NULL, info, theta))
 * whose input X is first refreshed from host memory: X_host (host, pinned
 * for overlap; n_local x d fp32 row-major) is copied into the device buffer
 * given to kmeans_create (which this call overwrites) in `chunks` row blocks
 * (clamped to [1, 64]) on a private copy stream, and the dense tensor-core
 * assignment starts on each block as soon as it has landed, so the transfer
 * overlaps the contraction. Other engines (SIMT, cfg.bounded) copy first,
 * then run the pass. Requires a started run (kmeans_aa_step with C0) and
 * cfg.x_refresh = 1 at create.  X_host's rows must lie inside the create-time
 * ranges of X (max |x_ik| and max ||x_i|| of the shard given to kmeans_create:
 * every operand scale and fixed-point scale was derived from them); a device
 * check after the copy enforces it, and a violation poisons the handle, reported
 * as INVALID by the next synchronising call (step info, kmeans_run).  The
 * bounded engine's per-row bounds are reset (new rows).
 * Asynchronous unless info/theta are requested; X_host must stay valid until
 * the stream has passed this call. Collective when nranks > 1. Errors: INVALID
 * for a NULL X_host with n_local > 0 or cfg.x_refresh = 0. */
AAKM_API kmeans_status kmeans_aa_step_host(kmeans_handle *h, const float *X_host /*host*/, int32_t chunks,
                                           kmeans_step_info *info /*host*/, double *theta_out /*host*/);

/* Per-pass trace of the Algorithm 1 run since its line 1 (kmeans_aa_step(C0) or
 * kmeans_run): one record per loop pass t = 1, 2, ... (the fields of
 * kmeans_step_info; the converged pass included), at most AAKM's device ring
 * of 8192 passes.  out: host, cap records (nullable when cap == 0); n_out:
 * host, the number of records the run holds (may exceed cap: the first cap are
 * copied).  Synchronises. */
AAKM_API kmeans_status kmeans_trace_export(kmeans_handle *h, kmeans_step_info *out /*host*/, int64_t cap,
                                           int64_t *n_out /*host*/);

/* Checked-workspace mode (test hook; compute-sanitizer is unavailable on the
 * GPU pool): with the environment variable AAKM_WS_CANARY=1 set before
 * kmeans_workspace_size / kmeans_create, every region of the workspace carve is
 * followed by a 256-byte canary (0xA5) written at create.  This call counts the
 * canary bytes that changed (a kernel wrote past the end of its region):
 * bad_bytes (host) must stay 0; n_guards (host, nullable) = canaries checked
 * (0 when the mode is off).  Synchronises. */
AAKM_API kmeans_status kmeans_debug_check_canaries(kmeans_handle *h, int64_t *bad_bytes /*host*/,
                                                   int64_t *n_guards /*host*/);

/* Sum of CUDA-event durations (ms) of the assignment launches recorded since
 * the last call (config.timing = 1), and their count.  Synchronises. */
AAKM_API kmeans_status kmeans_assign_timing(kmeans_handle *h, double *ms_total /*host*/,
                                   int64_t *launches /*host*/);

/* The same for the update partials of those G-evaluations (the label-sorted
 * segmented sums with the energy, or the atomic engine), branch A only.
 * Synchronises. */
AAKM_API kmeans_status kmeans_update_timing(kmeans_handle *h, double *ms_total /*host*/,
                                   int64_t *launches /*host*/);

/* Number of library kernels launched on this handle so far (graph replays
 * count every kernel node). */
AAKM_API int64_t kmeans_launch_count(const kmeans_handle *h);

/* Rows flagged as near-ties (re-decided in fp64) by the last assignment. */
AAKM_API kmeans_status kmeans_last_flagged(kmeans_handle *h, int64_t *flagged /*host*/);

/* Assignment work since the last Algorithm 1 line 1 (kmeans_aa_step(C0) /
 * kmeans_run): rows run through the assignment engine vs rows assigned
 * (local to this rank).  Equal unless cfg.bounded proved rows unchanged. */
AAKM_API kmeans_status kmeans_bounded_stats(kmeans_handle *h, int64_t *rows_scored /*host*/,
                                            int64_t *rows_total /*host*/);

/* Update work of this rank since the last Algorithm 1 line 1 (label-sorted
 * engine, plain combine; zeros otherwise): G-evaluations, how many took the
 * incremental update S(P^t) = S(P^{t-1}) + the moved rows (exact: bitwise the
 * full sums; chosen on the device, per rank, when at most n_local /
 * AAKM_DELTA_DIV (64) of the rank's rows moved; S_ref is the rank's own partial,
 * allreduced out of place), and the rows those moved. */
AAKM_API kmeans_status kmeans_update_stats(kmeans_handle *h, int64_t *n_evals /*host*/,
                                           int64_t *n_incremental /*host*/, int64_t *rows_moved /*host*/);

/* Exactness-margin probe (test hook): runs the handle's dense assignment
 * engine on C (K x d fp64) and writes, per local row, the engine's raw top-2
 * values and its near-tie threshold: rows_out (device, n_local x 4 float) =
 * (b1, b2, tau, bits of the chosen index i1), before any near-tie refine.
 * kind_out (host): 1 = a tensor-core engine (3xTF32 or 2xFP16), values are
 * window accumulators U ||x - c||^2 + 6 with U = *unit_out (host, 1/(2 s^2));
 * 2 = SIMT FP32, values are scores ||c||^2 - 2 x.c (unit 1).  (0 is no longer
 * produced: r01's 3xTF32 key-packed scores.)  Every computed value must lie within tau / 2 of
 * its exact counterpart for the near-tie flagging (row a3) to be rigorous.
 * Synchronises; clobbers the API label buffer only. */
AAKM_API kmeans_status kmeans_debug_scores(kmeans_handle *h, const double *C, float *rows_out,
                                           int32_t *kind_out /*host*/, double *unit_out /*host*/);

/* Bounded engine (cfg.bounded) test hooks.
 * export: the Hamerly state between passes -- per local row ub (upper bound on
 * ||x_i - c_ref,rho_i||, and on the second candidate's distance when p2 >= 0),
 * lb (lower bound on every other ||x_i - c_ref,j||), p2 (the two-centroid row's
 * other candidate, -1 if none) -- and C_ref (K x d fp64, the centroid set the
 * bounds refer to); rho_i are the labels of the last assignment (state export's
 * labels_prev).  Device outputs, each nullable.  Synchronises.
 * repeat: runs the bounded assignment of the current iterate twice back to back
 * (the second call sees zero drift), writes the bounds after the first call
 * (device, nullable), the rows each call re-scored on the tensor engine
 * (scored_out, host 2) and whether the labels agree (same_out, host).
 * DESTRUCTIVE (overwrites P^{t-1}); restart with kmeans_aa_step(C0).
 * Errors: INVALID without a bounded engine; STATE outside a live run. */
AAKM_API kmeans_status kmeans_bounds_export(kmeans_handle *h, float *ub_out, float *lb_out, int32_t *p2_out,
                                            double *Cref_out);
AAKM_API kmeans_status kmeans_bounds_repeat(kmeans_handle *h, float *ub1_out, float *lb1_out,
                                            int64_t *scored_out /*host*/, int32_t *same_out /*host*/);

/* How the ranks combine: mode (host) = -1 no communicator, 0 ncclAllReduce,
 * 1 fused multimem (NVLS), 2 fused LSA unicast; lsa_size (host, nullable) =
 * ranks in the NVLink team of the fused path (0 otherwise). */
AAKM_API kmeans_status kmeans_comm_info(kmeans_handle *h, int32_t *mode /*host*/, int32_t *lsa_size /*host*/);

/* Name of the assignment engine the handle selected ("simt"/"tc"/"tc16"). */
AAKM_API const char *kmeans_assign_path_name(const kmeans_handle *h);

AAKM_API kmeans_status kmeans_destroy(kmeans_handle *h);

/* Last error message of h (NULL h: this thread's last create error). */
AAKM_API const char *kmeans_last_error(const kmeans_handle *h);

AAKM_API int32_t kmeans_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* AAKM_H */
