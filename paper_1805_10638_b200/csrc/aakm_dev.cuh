// aakm_dev.cuh -- internal declarations shared by the sm_100a kernels and the
// host runtime of libaakm.so.  Not part of the ABI (see include/aakm.h).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define AAKM_H_SLOTS 32           // ring capacity >= m_max + 1 (KMEANS_M_MAX = 30)
#define AAKM_UPD_MAX_BLOCKS 1184  // 8 x 148 SMs
#define AAKM_GRAM_BLOCKS 148
#define AAKM_TRACE_CAP 8192
#define AAKM_MAXC 32               // candidates kept per flagged row
#define AAKM_SORTED_MIN_ROWS 65536  // label-sorted update engine from this many rows
#define AAKM_PRIV_MAX_KD 4096       // ... whose S/N fit one block's shared memory (2 K d + K int32)
#define AAKM_PRIV_MAX_ROWS (1 << 18) // and shards small enough that one kernel beats sort + segmented sums
#define AAKM_SORTED_MAX_K 16384     // ... and up to this many clusters (smem histograms)
#define AAKM_SEG_BLOCKS_MAX 512     // row blocks of the histogram / scatter (Dev::seg_blocks)
#define AAKM_MAX_RANKS 1024         // NCCL ranks per communicator this build sizes for
#define AAKM_SEED_BLOCKS 1184      // row blocks of the K-Means++ passes (8 x 148)
#define AAKM_MAX_LSA 8              // f4 unicast fallback: LSA peers (one NVLink domain of 8 GPUs)
#define AAKM_CNIMG_BYTES 4096       // folded ||c||^2 block of one 128-centroid tile (128 rows x 32 B)

namespace aakm {

// Per-pass trace record (host-readable through kmeans_step_info / report).
struct TraceRec {
    long long t, changed;
    double E_cand, E_final;
    int m, m_t, accepted, rejected, converged, lloyd;
};

// Device-resident Algorithm 1 control state.  Every
// decision is taken on the device from allreduced scalars, so all ranks take
// identical branches and the host never round-trips inside a pass.
struct alignas(16) DevState {
    long long t;                 // pass index of the current iterate C^t
    long long n_accepted, n_rejected, n_assign;
    long long changed;           // #changed labels of the final P^t
    long long last_flag[2];      // near-tie rows of the last assignments A / B (diagnostics)
    long long trace_len;
    double E1, E2;               // E^{t-1}, E^{t-2}, post-guard (R-A7)
    double E_cand, E_final;      // E^t before / after the guard
    int m, m_t, lloyd, reject;
    int done, converged, cur, init_mode;
    int hist_count, accepted_now, rejected_now, label_error;
    int n_alpha, fb_slot, final_traced, pad0;
    unsigned int cmax2_bits;     // max_j ||c_j||^2 of the centroids being assigned (float bits)
    unsigned int cmax2_tmp, comb_ctr, upd_ctr, hist_ctr;
    float c_scale;               // 2xFP16 engine: common power-of-two operand scale s (x/s, c/s)
    float tau_abs;               // 2xFP16 engine: absolute term of the near-tie bound
    float cn_amul;               // 2xFP16 engine: power-of-two A-side factor of the folded ||c||^2 column
    unsigned int x_amax_bits;    // create-time scratch: max |x| over the shard (2xFP16 X scale)
    int bnd_ready, bnd_use;      // bounded engine: bounds valid for the next / this assignment
    long long rows_scored, rows_total;   // bounded engine: rows run through the tensor engine / all rows
    unsigned int shift_max_bits, shift_tmp, shift_ctr, pad3;   // max_j ||c_j - c_ref_j|| (float bits)
    long long seed_max;          // K-Means++: max_i D2_i of the current round (fixed point)
    int seed_err, pad4;          // K-Means++: 2 = fewer distinct samples than K
    int bnd_ready0, pad5;        // bounded engine: bnd_ready at the snapshot
    unsigned int fc_ctr, pad6;   // f4 fused combine: blocks done zeroing (comm.cu)
    int sref_valid, use_delta;   // incremental update: S_ref = S(P^{t-1}) valid / this evaluation uses it
    unsigned int delta_ctr, pad7;
    long long n_upd, n_delta, rows_moved;   //   evaluations / of them incremental / their moved rows
    double theta[AAKM_H_SLOTS];
    double alpha[AAKM_H_SLOTS];
    int alpha_slot[AAKM_H_SLOTS];
    double gram[AAKM_H_SLOTS * AAKM_H_SLOTS];  // <dF(tau_a), dF(tau_b)>, slot-indexed (tau mod H)
    double bvec[AAKM_H_SLOTS];                 // <dF(t-j+1), F^t>, j = 1..W
};

// Everything a kernel needs, passed by value.
struct Dev {
    const float* X;       // n x d samples (borrowed)
    long long n;          // local rows
    int d, K, H, m_max, m0, dynamic_m;
    long long max_iters;
    double eps1, eps2, ridge;
    DevState* st;
    double* C;            // current iterate C^t (K x d, fp64: the Anderson state is fp64, R-A17)
    float* C32;           // fl32(C^t): the SIMT engine's operand (its bound adds |c - fl32(c)|)
    float* Chi;           // tf32(-C) (tensor path)
    float* Clo;           // -C - tf32(-C) rounded to fp32
    float* cn;            // ||c_j||^2 (fp32, from fp64)
    uint8_t* cnimg;       // tensor engines: ||c||^2/2 column block per 128-centroid tile, UMMA
                          // no-swizzle K-major image (AAKM_CNIMG_BYTES per tile); nullptr on SIMT
    unsigned int key_mul; // 32, from the host (keeps the key pack on the FMA pipe, see assign_tc.cu)
    void* Chi16;          // 2xFP16 engine: fp16 hi of C / s_c
    void* Clo16;          // 2xFP16 engine: fp16 lo
    int tc_kind;          // 0 = 3xTF32, 1 = 2xFP16
    int pair_ok;          // two-centroid near-tie fast path (k_refine_pair: d/4 a power of two <= 32)
    float x_scale;        // 2xFP16: create-time scale from max |x| (informational)
    float x_inv_scale;
    float x_absmax;       // 2xFP16: max |x_ik| over the shard (subnormal part of the error bound)
    float x_nmax;         // 2xFP16: max ||x_i|| over the shard (fixes the common operand scale)
    int* lab[2];          // label ping-pong, lab[cur] = P^t, lab[cur^1] = P^{t-1}
    int* flag_rows;       // near-tie row list (capacity n)
    float* flag_b1;       // best fp32/3xTF32 score of each flagged row (capacity fcap)
    float* flag_tau;      // its gap threshold tau_i
    float* Xf;            // gathered flagged rows (fcap x d) for the candidate pass
    int* cand;            // candidate centroids per flagged row (fcap x AAKM_MAXC)
    int* cand_cnt;        // candidate counts per flagged row and epilogue half (> AAKM_MAXC/2 = overflow)
    long long fcap;       // capacity of the candidate path (rows beyond -> SIMT refine)
    long long* flag_count;// [2] near-tie counts of branch A / B (zeroed per pass with packed)
    int* pair_rows;       // near-tie rows whose window holds exactly two centroids (capacity fcap)
    int2* pair_j;         //   their two centroids (best key, runner-up)
    long long* pair_count;//   [2] counts, branch A / B (zeroed per pass with the flags)
    long long* delta_count;// [2] incremental update: moved rows of branch A / B (zeroed likewise)
    long long* packed[2]; // [S_hi (K*d) | S_lo (K*d) | N (K) | E_hi | E_lo | E (fp64 bits) | changed | X2_hi | X2_lo]
    float fx_scale;       // 2^(22-e), |x| <= 2^e over all ranks: S in exact fixed point (update.cu)
    double fx_inv;        // 2^(e-22)
    double xn_gmax;       // max_i ||x_i|| over all ranks (rounded up): bounds every ||x_i - c||
    long long* sref;      // incremental update (sorted engine): this rank's [S_hi | S_lo | N] of P^{t-1}
    long long* partial[2];// where the update kernels add this rank's contributions: packed[b]
                          // itself, or (incremental update with a communicator) a local buffer
                          // that the allreduce reads (out of place) -- S_ref is a LOCAL partial
                          //   (nullptr: off); k_finalize writes it, k_delta_* read it
    long long delta_max;  //   at most this many moved rows take the incremental path
    long long* x2;        // sorted engine: this rank's sum_i ||x_i||^2 in units of 2^x2_e (two parts, as
    int x2_e;             //   energy_flush), refreshed with X; x2_e = frexp exponent of 2 xn_gmax^2 - 51
    double* upd_part;     // per-block (E, changed) partials
    int* seg_bh;          // sorted update engine: per-block histograms -> scatter bases (SEG_BLOCKS x K)
    int* seg_off;         // row offsets of cluster j in perm (K+1)
    int* seg_chunk;       // chunk offsets (K+1)
    long long* seed_d2;   // K-Means++: D2_i (n, fixed point, seed.cu)
    int* seed_near;       // K-Means++: index of a chosen center at D2_i from row i (n)
    double* seed_cc;      // K-Means++: lower bounds of ||c_q - c_j||, j < q, for the newest center q (K)
    long long* seed_part; // K-Means++: per-block weight sums (AAKM_SEED_BLOCKS)
    long long* seed_T;    // K-Means++: every rank's weight total (nranks)
    int* seed_x;          // K-Means++: exchange row (d fp32 bits + global index)
    long long* seed_idx;  // K-Means++: chosen global indices (K)
    double* seed_u;       // K-Means++: the caller's uniforms (K)
    const void* xg_map;   // device copy of the gather4 map of X (nullptr: generic segmented sums)
    int4* seg_cmap;       // chunk -> {cluster j, first sorted row, rows, 0} (n/SEG_ROWS + K)
    int* perm;            // rows bucketed by label (n)
    float* ub;            // bounded engine (nullptr = dense): per row, upper bound on ||x_i - c_{rho_i}||
    float* lb;            //   ... and lower bound on min_{j != rho_i} ||x_i - c_j||, w.r.t. C_ref
    int* pj2;             //   two-centroid rows: the other candidate (-1: none); then ub bounds
                          //   both candidates' distances and lb every other centroid's
    float* pgap;          //   two-centroid rows: lower bound on d(x, c_other) - d(x, c_label)
                          //   from the last exact decision, moved by the shifts (w.r.t. C_ref)
    int* act_rows;        //   rows the bounds could not prove unchanged (capacity n)
    long long* act_count; //   [2] their counts, branch A / B (zeroed per pass with packed)
    double* C_ref;        //   centroids the bounds refer to (the last assigned set)
    float* shift;         //   ||c_j - c_ref_j|| of the set being assigned (K)
    float* ub0;           //   snapshot of (ub, lb, pj2, C_ref) taken before branch A, restored
    float* lb0;           //   for the fallback B on a rejection (bounds w.r.t. the previous
    int* pj20;            //   pass's set instead of the rejected jump)
    float* pgap0;
    double* C_ref0;
    double* Gring;        // H x K*d (fp64)
    double* Fring;        // H x K*d (fp64)
    double* gram_part;    // AAKM_GRAM_BLOCKS x (2*H)
    TraceRec* trace;
    int nranks;
    int upd_blocks;
    int upd_sorted;       // label-sorted update engine (chosen from n_global, d, K: the same on every rank)
    int upd_priv;         // small K*d shards of the sorted engine: one kernel, S/N in shared memory
    int seg_blocks;       // its row blocks (histogram / scatter partition; 2 per SM for K <= 4096)
    int gram_blocks;
    float tau_gamma;      // near-tie threshold factor of the active assignment engine
    int dbg;              // AAKM_TC_DBG probe bits (perf experiments only; 0 in normal runs)
    float4* dbg_rows;     // kmeans_debug_scores only: per row (b1, b2, tau, i1 bits) of the dense engine
    unsigned long long* dbg_ts;   // AAKM_TC_TRACE probe: pipeline event stamps (nullptr in normal runs)
    unsigned long long condB;     // kmeans_run's CUDA graph: conditional handle of the fallback branch B
                                  // (k_control sets it on a rejection; 0 = eager launches, no conditional)
    // f4 fused combine (cfg.fused_comm, comm.cu): packed[0] / packed[1] are this rank's
    // replica of an NCCL symmetric window; every flush adds into all replicas
    int fused;            // 0 off, 1 multimem (NVLS multicast address mc0), 2 LSA peer pointers
    int lsa_n;            // LSA peers (fused == 2), this rank included
    long long pk_off1;    // words from packed[0] to packed[1] inside the window
    long long* mc0;       // multicast address of packed[0]
    long long* lsa0[AAKM_MAX_LSA];   // every LSA peer's replica of packed[0]
    int dev;              // CUDA device ordinal of the handle
    int num_sms;          // its SM count (persistent grids)
};
#define AAKM_MAX_DEVICES 64

// Which labels/centroids a G-evaluation kernel works on.
struct GEval {
    int branch;           // 0 = candidate C^t, 1 = fallback C_AU^t (predicated on reject)
    int force;            // 1 = run regardless of done/reject (API calls)
    int* lab_out;         // nullptr -> d.lab[st->cur]
    const int* lab_prev;  // used when prev_mode == 2
    int prev_mode;        // 0 = d.lab[st->cur ^ 1], 1 = none, 2 = lab_prev
    long long* packed_out;// nullptr -> d.packed[branch]
    long long tile0, tile1;  // MODE 0 dense engine: row tiles [tile0, tile1) only (tile1 = 0: all)
};

__device__ __forceinline__ bool geval_active(const Dev& d, const GEval& g) {
    if (g.force) return true;
    const volatile DevState* st = d.st;
    if (st->done) return false;
    return g.branch == 0 || st->reject;
}

// ---- launchers (host side, defined in the .cu files) ----
void launch_combine(const Dev& d, int mode, const double* src, cudaStream_t s);
void launch_assign_simt(const Dev& d, const GEval& g, cudaStream_t s);
void launch_assign_tc(const Dev& d, const GEval& g, const void* maps, cudaStream_t s);
void* tc_make_maps(const Dev& d);   // TMA tensor maps of (X, C_hi, C_lo); nullptr if unsupported
void tc_free_maps(void* m);
// 128-byte TMA map of X (n x d fp32) with a {d, 1} box for tile::gather4 row gathers
// (the update's segmented sums); false if d is not a multiple of 4 in [4, 128].
bool encode_gather_rows(void* map128, const float* X, long long n, int d);
// K-Means++ seeding (seed.cu)
cudaError_t setup_seed();
int seed_blocks(const Dev& d);
void launch_seed_first(const Dev& d, long long row_local, long long gi, cudaStream_t s);
int launch_seed_dist(const Dev& d, const float* C, int q, double scale, cudaStream_t s);   // launches
void launch_seed_weights(const Dev& d, int log2n, int rank, int nranks, cudaStream_t s);
void launch_seed_select(const Dev& d, int r, int log2n, int rank, int nranks, long long row_offset, cudaStream_t s);
void launch_seed_commit(const Dev& d, float* C_out, int r, cudaStream_t s);
bool tc_supported(int d, int K);
bool tc16_supported(int d, int K);
float tau_gamma_tc16(int d);
void launch_csplit16(const Dev& d, int mode, cudaStream_t s);
int launch_bounds_prep(const Dev& d, const GEval& g, cudaStream_t s);   // k_shift + k_bounds
void launch_assign_tc_bounded(const Dev& d, const GEval& g, const void* maps, cudaStream_t s);
__host__ __device__ inline unsigned int cnimg_off(int r, int byte) {   // (row, byte in its 32-B K row)
    return (unsigned)((r >> 3) * 256 + (byte >> 4) * 128 + (r & 7) * 16 + (byte & 15));
}
// the launchers below return how many kernels they enqueued (the gpu_launches count)
int launch_refine(const Dev& d, const GEval& g, cudaStream_t s, long long first = 0);
int launch_refine_tc(const Dev& d, const GEval& g, const void* maps, cudaStream_t s);
int launch_update(const Dev& d, const GEval& g, cudaStream_t s);
bool update_sorted(long long n_global, int dd, int K);
int seg_blocks_for(int K, int num_sms);
void launch_control(const Dev& d, int stage, cudaStream_t s);
void launch_finalize(const Dev& d, cudaStream_t s);
void launch_gram(const Dev& d, cudaStream_t s);
void launch_solve(const Dev& d, cudaStream_t s);
void launch_advance(const Dev& d, cudaStream_t s);
void launch_reset(const Dev& d, cudaStream_t s);
void launch_update_G(const Dev& d, const long long* packed, const double* Cprev, double* G,
                     long long* counts, cudaStream_t s);
void launch_energy(const Dev& d, const GEval& g, cudaStream_t s);       // E after the allreduce
// sorted engine: E's parts from the (reduced or local) packed S, N, X2 and C (update.cu)
int launch_energy_x(const Dev& d, const GEval& g, cudaStream_t s);
void launch_partials_out(const Dev& d, const long long* packed, double* out, cudaStream_t s);
// (x2: also sum_i ||x_i||^2 as launch_x2, in the same pass when d = 4 LPR); returns launches
int launch_xstats_max(const float* X, long long n, int d, unsigned int* out, cudaStream_t s,
                      long long* x2 = nullptr, int x2_e = 0);
// sum_i ||x_i||^2 of the shard (count = n d floats) in units of 2^x2_e, two parts into out[2] (zeroed)
void launch_x2(const float* X, long long count, int x2_e, long long* out, cudaStream_t s);
// f4 fused combine (comm.cu); comm is an ncclComm_t; setup returns an error message or nullptr
const char* fused_setup(void** handle, void* comm, Dev& d, void* scratch, cudaStream_t s);
void fused_free(void* handle, void* comm);
int fused_mode(const void* handle);
int fused_lsa_size(const void* handle);
int launch_fused_zero(const Dev& d, const GEval& g, const void* handle, cudaStream_t s);
int launch_fused_flushed(const Dev& d, const GEval& g, const void* handle, cudaStream_t s);
// st->label_error |= 2 if the stats in out (launch_xstats_max) exceed (amax, nmax2) (float bits)
void launch_xcheck(const Dev& d, const unsigned int* out, unsigned int amax, unsigned int nmax2, cudaStream_t s);

// fixed-point sums (update.cu) -> fp64: (hi + lo 2^-22) 2^(e-22), exact conversions
__host__ __device__ inline double fx_value(long long hi, long long lo, double fx_inv) {
    return ((double)hi + (double)lo * 2.384185791015625e-07) * fx_inv;
}
// packed-vector word offsets
__host__ __device__ inline long long pk_n(const Dev& d) { return 2LL * d.K * d.d; }           // N_j at + j
__host__ __device__ inline long long pk_ehi(const Dev& d) { return 2LL * d.K * d.d + d.K; }   // E_hi, E_lo
__host__ __device__ inline long long pk_e(const Dev& d) { return pk_ehi(d) + 2; }             // E (fp64 bits)
__host__ __device__ inline long long pk_ch(const Dev& d) { return pk_ehi(d) + 3; }            // changed
__host__ __device__ inline long long pk_x2(const Dev& d) { return pk_ehi(d) + 4; }            // X2_hi, X2_lo
__host__ __device__ inline long long pk_words(const Dev& d) { return pk_ehi(d) + 6; }
// Energies e_i = ||x_i - c_rho_i||^2 go into the packed vector as a two-part fixed
// point [E_hi (units 1/q) | E_lo (units 2^-30/q)]. q = 2^(21 - eb) with
// 2^eb > B = 2 (max||x|| + max||c||)^2 >= every e_i, so any partial e of one row
// scales to v = e q < 2^21; energy_fx rounds v to a multiple of 2^-30 (adding
// 1.5*2^22, whose ulp is 2^-30, rounds exactly) and returns it as an integer < 2^51.
// A lane sums at most 256 of them in an int64 (< 2^59) and moves the sum into the
// two parts with energy_flush. Each partial carries 2^-52 of B; an exact 0 stays 0;
// the integer sums do not depend on order.
__device__ inline double energy_q(const Dev& d) {
    const double cm = sqrt((double)__uint_as_float(d.st->cmax2_bits));
    const double B = 2.0 * (d.xn_gmax + cm) * (d.xn_gmax + cm);
    int eb = 0;
    frexp(B > 0.0 ? B : 1.0, &eb);
    return ldexp(1.0, 21 - eb);
}
__device__ inline long long energy_fx(double v) {
    return __double_as_longlong(v + 6291456.0) - 0x4158000000000000LL;
}
// the same before the constant is removed (the caller subtracts count * ENERGY_FX_BIAS
// once per flush): energy_bits(e, q) - ENERGY_FX_BIAS == energy_fx(e * q) (q is a power of 2)
#define ENERGY_FX_BIAS 0x4158000000000000LL
__device__ inline long long energy_bits(double e, double q) { return __double_as_longlong(fma(e, q, 6291456.0)); }
__device__ inline void energy_flush(long long& acc, long long& hi, long long& lo) {
    hi += acc >> 30;
    lo += acc & 0x3fffffffLL;
    acc = 0;
}

// ---- programmatic dependent launch (PDL) for the latency-bound kernels of a pass.
// A kernel launched through launch_pdl may be scheduled while its predecessor in the
// stream is still running; its FIRST statement is pdl_wait() (griddepcontrol.wait:
// blocks until the predecessor grid completed and its writes are visible; a no-op
// when the launch had no programmatic dependency), so nothing it reads can be stale.
// pdl_trigger() lets the successor's launch begin early.  g_pdl (AAKM_PDL, default
// on) switches the attribute off for A/B runs.
extern int g_pdl;
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid; cfg.blockDim = block; cfg.dynamicSmemBytes = smem; cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = g_pdl ? 1 : 0;
    cfg.attrs = at; cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}

// one-time kernel attribute setup (max dynamic smem); never during stream capture
cudaError_t setup_simt();
cudaError_t setup_refine();
cudaError_t setup_update();
cudaError_t setup_tc();

// error-bound factors of the two engines
float tau_gamma_simt(int d);
float tau_gamma_tc(int d);

}  // namespace aakm
