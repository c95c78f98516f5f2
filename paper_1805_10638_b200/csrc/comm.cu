// comm.cu -- f4: the cross-rank combine of row a7 fused into the
// update's flushes through NCCL 2.28's device API (cfg.fused_comm).
//
// Plain path: every rank red.adds its partials into a private packed vector
// [S_hi | S_lo | N | E_hi | E_lo | E | changed] (exact int64 fixed point) and
// one ncclAllReduce(sum, int64) per G-evaluation combines them.
//
// Fused path: the two packed vectors (branch A / B) live in an NCCL symmetric
// window (ncclMemAlloc + ncclCommWindowRegister, NCCL_WIN_COLL_SYMMETRIC), and
// every flush of the update kernels (update.cu pk_add) adds into ALL ranks'
// replicas at once:
//   mode 1  multimem.red.relaxed.sys.global.add.u64 on the window's LSA
//           multicast address: one NVLink transaction per flushed word, the
//           NVSwitch applies the add to every replica (NVLS);
//   mode 2  (no multicast object, e.g. a single rank) red.relaxed.sys.global.add
//           into each LSA peer's replica through its peer pointer (P2P stores).
// Protocol per G-evaluation (all ranks take identical branches: the control is
// replicated), with two LSA device barriers (ncclLsaBarrierSession, acq_rel at
// system scope) instead of a collective launch:
//   k_fc_zero     zero this rank's replica of the branch's buffer, then barrier 0
//                 ("zeroed"): no rank adds into a replica before its owner reset it
//   update        hist / scans / scatter / segmented sums: pk_add into all replicas
//   k_fc_flushed  barrier 1 ("flushed"): every rank's adds have landed everywhere
// after which k_energy / k_control / k_finalize read the local replica as before.
// Integer adds are associative and exact, so every replica holds the same bytes
// as the allreduce path (for any rank count); tests/test_gpu_fused.py checks it.
#include <nccl.h>
#include <nccl_device.h>

#include "aakm_dev.cuh"

namespace aakm {

__global__ void k_fc_ptrs(const __grid_constant__ ncclDevComm dc, ncclWindow_t win, int mm, long long** out) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    out[0] = mm ? reinterpret_cast<long long*>(ncclGetLsaMultimemPointer(win, 0, dc)) : nullptr;
    for (int r = 0; r < AAKM_MAX_LSA; ++r)
        out[1 + r] = r < dc.lsaSize ? reinterpret_cast<long long*>(ncclGetLsaPointer(win, 0, r)) : nullptr;
    out[1 + AAKM_MAX_LSA] = reinterpret_cast<long long*>((long long)dc.lsaSize);
}

__device__ __forceinline__ void fc_barrier(const ncclDevComm& dc, int index, bool mm) {
    __threadfence_system();
    ncclLsaBarrierSession<ncclCoopThread> bar(ncclCoopThread(), dc, ncclTeamTagLsa(), (uint32_t)index, mm);
    bar.sync(ncclCoopThread(), cuda::memory_order_acq_rel);
    __threadfence_system();
}

// zero the local replica of this branch's buffer (all blocks), then -- once every
// block is done (last-block counter) -- the "zeroed" barrier
__global__ void __launch_bounds__(256) k_fc_zero(Dev d, GEval g, const __grid_constant__ ncclDevComm dc, long long words) {
    if (!geval_active(d, g)) return;
    long long* buf = d.packed[g.branch];
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < words; i += (long long)gridDim.x * blockDim.x)
        buf[i] = 0;
    __threadfence_system();
    __syncthreads();
    __shared__ bool last;
    if (threadIdx.x == 0) last = atomicAdd(&d.st->fc_ctr, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last || threadIdx.x != 0) return;
    d.st->fc_ctr = 0;
    fc_barrier(dc, 0, d.fused == 1);
}

__global__ void k_fc_flushed(Dev d, GEval g, const __grid_constant__ ncclDevComm dc) {
    if (!geval_active(d, g)) return;
    if (threadIdx.x == 0) fc_barrier(dc, 1, d.fused == 1);
}

struct FusedComm {
    void* buf = nullptr;
    size_t bytes = 0;
    ncclWindow_t win = nullptr;
    ncclDevComm dc;
    bool have_dc = false;
    int mode = 0;
};

// Collective (every rank, same order).  On success d gets the window buffers as
// packed[0] / packed[1] and the multicast / peer addresses; returns a message on error.
const char* fused_setup(void** handle, void* comm_v, Dev& d, void* scratch, cudaStream_t s) {
    ncclComm_t comm = static_cast<ncclComm_t>(comm_v);
    FusedComm* f = new FusedComm();
    *handle = f;
    const size_t pkb = ((size_t)pk_words(d) * 8 + 4095) & ~(size_t)4095;
    f->bytes = 2 * pkb;
    if (ncclMemAlloc(&f->buf, f->bytes) != ncclSuccess) return "ncclMemAlloc failed";
    if (cudaMemsetAsync(f->buf, 0, f->bytes, s) != cudaSuccess) return "cudaMemsetAsync(window) failed";
    if (ncclCommWindowRegister(comm, f->buf, f->bytes, &f->win, NCCL_WIN_COLL_SYMMETRIC) != ncclSuccess)
        return "ncclCommWindowRegister failed";
    const char* force = getenv("AAKM_FUSED_MODE");                 // 2: force the unicast path
    for (int mm = (force && atoi(force) == 2) ? 0 : 1; mm >= 0; --mm) {
        ncclDevCommRequirements reqs;
        memset(&reqs, 0, sizeof(reqs));
        reqs.lsaBarrierCount = 2;
        reqs.lsaMultimem = mm != 0;
        if (ncclDevCommCreate(comm, &reqs, &f->dc) == ncclSuccess) { f->have_dc = true; f->mode = mm ? 1 : 2; break; }
    }
    if (!f->have_dc) return "ncclDevCommCreate failed";
    long long** dptr = static_cast<long long**>(scratch);          // >= (AAKM_MAX_LSA + 2) pointers, free at create
    k_fc_ptrs<<<1, 32, 0, s>>>(f->dc, f->win, f->mode == 1, dptr);
    long long* hp[AAKM_MAX_LSA + 2];
    const cudaError_t e = cudaMemcpyAsync(hp, dptr, sizeof(hp), cudaMemcpyDeviceToHost, s);
    const cudaError_t e2 = cudaStreamSynchronize(s);
    if (e != cudaSuccess || e2 != cudaSuccess) return "window address query failed";
    const int lsa = (int)(long long)hp[1 + AAKM_MAX_LSA];
    if (f->mode == 2 && lsa > AAKM_MAX_LSA) return "fused_comm unicast path supports <= 8 LSA peers";
    if (f->mode == 1 && !hp[0]) return "no multicast address for the window";
    d.fused = f->mode;
    d.lsa_n = lsa < AAKM_MAX_LSA ? lsa : AAKM_MAX_LSA;
    d.mc0 = hp[0];
    for (int r = 0; r < AAKM_MAX_LSA; ++r) d.lsa0[r] = hp[1 + r];
    d.pk_off1 = (long long)(pkb / 8);
    d.packed[0] = reinterpret_cast<long long*>(f->buf);
    d.packed[1] = reinterpret_cast<long long*>(reinterpret_cast<char*>(f->buf) + pkb);
    d.partial[0] = d.packed[0]; d.partial[1] = d.packed[1];   // the flushes add into the window itself
    return nullptr;
}

int fused_mode(const void* handle) { return handle ? static_cast<const FusedComm*>(handle)->mode : 0; }
int fused_lsa_size(const void* handle) {
    const FusedComm* f = static_cast<const FusedComm*>(handle);
    return f && f->have_dc ? f->dc.lsaSize : 0;
}

void fused_free(void* handle, void* comm_v) {
    ncclComm_t comm = static_cast<ncclComm_t>(comm_v);
    FusedComm* f = static_cast<FusedComm*>(handle);
    if (!f) return;
    if (comm && f->have_dc) ncclDevCommDestroy(comm, &f->dc);
    if (comm && f->win) ncclCommWindowDeregister(comm, f->win);
    if (f->buf) ncclMemFree(f->buf);
    delete f;
}

int launch_fused_zero(const Dev& d, const GEval& g, const void* handle, cudaStream_t s) {
    const FusedComm* f = static_cast<const FusedComm*>(handle);
    const long long words = pk_words(d);
    int blocks = (int)((words + 255) / 256);
    if (blocks > 2 * d.num_sms) blocks = 2 * d.num_sms;
    if (blocks < 1) blocks = 1;
    k_fc_zero<<<blocks, 256, 0, s>>>(d, g, f->dc, words);
    return 1;
}

int launch_fused_flushed(const Dev& d, const GEval& g, const void* handle, cudaStream_t s) {
    const FusedComm* f = static_cast<const FusedComm*>(handle);
    k_fc_flushed<<<1, 32, 0, s>>>(d, g, f->dc);
    return 1;
}

}  // namespace aakm
