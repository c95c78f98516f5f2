// assign_tc.cu -- tcgen05/TMEM 3xTF32 assignment engine (sm_100a).
//
// Assignment step, Eq. (3), through the expansion
// ||x||^2 - 2 x.c + ||c||^2 (north_star): the sample-centroid contraction
// X C^T is a dense GEMM (M = rows, N = centroids, K = d) run on the 5th-gen
// tensor cores with a 3xTF32 split so the dot products keep ~fp32 accuracy:
//     x.c ~= x_lo.c_hi + x_hi.c_lo + x_hi.c_hi,
//     hi = tf32(v) (low 13 mantissa bits cleared), lo = v - hi (exact in fp32).
// The argmin over centroids is fused into the epilogue (TMEM -> registers):
// per row the best score b1 (index i1, lowest index on fp32 ties) and the
// runner-up b2; rows with b2 - b1 within the engine's error bound are
// flagged for the exact fp64 re-decision in refine.cu.
//
// Persistent, warp-specialised CTA (one per SM), BM = 128 rows, BN = 128
// centroids per tile, UMMA 128 x 128 x 8 (kind::tf32, cta_group::1):
//   warp 0     TMA producer: X tile (once per row tile, SWIZZLE_128B) and a
//              ring of S stages, each one 32-element K-atom of C_hi and C_lo
//   warp 1     MMA issuer (one elected thread), accumulators in TMEM,
//              double-buffered (2 x 128 fp32 columns)
//   warp 2     TMEM allocator
//   warps 4-7  epilogue: split the X tile into hi/lo in shared memory,
//              then per tile tcgen05.ld 32 columns at a time, score, argmin
// X is read from HBM once; C tiles stream from L2.
#include <cuda.h>
#include <stdio.h>

#include "aakm_dev.cuh"

namespace aakm {

constexpr int TC_BM = 128;
constexpr int TC_BN = 128;
constexpr int TC_THREADS = 256;
constexpr int ATOM_BYTES_X = TC_BM * 128;          // one 32-element K-atom of the X tile
constexpr int STAGE_BYTES = 2 * TC_BN * 128;       // C_hi atom + C_lo atom
constexpr int SMEM_LIMIT = 232448;                 // 227 KB opt-in

// Error bound of the 3xTF32 scores: per-product split
// error <= 3 * 2^-20 |x_k c_k|; tensor-core fp32 accumulation over the
// 3d/8 MMA k-steps (+8 for the internal 8-term dot) at <= 2^-22 each.
// Both scores of the top-2 gap carry it, and ||x||^2 + max||c||^2 bounds
// 2 sum |x_k c_k|; factor 4 is the safety margin.
float tau_gamma_tc(int d) { return 4.0f * (3.0f * 9.5367432e-7f + (3.0f * d / 8.0f + 8.0f) * 2.3841858e-7f); }

struct TcMaps {
    CUtensorMap x, chi, clo, xf;
};

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t cnt) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(cnt) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
// Bounded wait: a lost arrival traps (error to the host) instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    uint32_t ok = 0;
    for (uint32_t spin = 0;; ++spin) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok) : "r"(su32(b)), "r"(parity) : "memory");
        if (ok) return;
        if (spin > (1u << 26)) __trap();
    }
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
        ::"r"(su32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(su32(bar)), "r"(c0), "r"(c1)
        : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// UMMA shared-memory descriptor: K-major, SWIZZLE_128B, 8-row core atoms of 1024 B.
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);        // start address (>> 4)
    d |= (uint64_t)1 << 16;                          // LBO (unused for swizzled K-major)
    d |= (uint64_t)(1024 >> 4) << 32;                // SBO: 8 rows x 128 B
    d |= (uint64_t)1 << 46;                          // descriptor version (sm_100)
    d |= (uint64_t)2 << 61;                          // SWIZZLE_128B
    return d;
}
// Instruction descriptor: D f32, A/B tf32, both K-major, M = 128, N = TC_BN.
constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(TC_BN >> 3) << 17) | ((uint32_t)(TC_BM >> 4) << 24);

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t accum) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
        ::"r"(tmem_d), "l"(a), "l"(b), "r"(IDESC), "r"(accum)
        : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar))
                 : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void push_flag_tc(const Dev& d, int branch, bool flag, long long row, float b1, float tau) {
    unsigned mask = __ballot_sync(0xffffffffu, flag);
    if (mask == 0) return;
    int lane = threadIdx.x & 31;
    int leader = __ffs(mask) - 1;
    long long base = 0;
    if (lane == leader)
        base = (long long)atomicAdd((unsigned long long*)&d.flag_count[branch], (unsigned long long)__popc(mask));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (flag) {
        const long long f = base + __popc(mask & ((1u << lane) - 1));
        d.flag_rows[f] = (int)row;
        if (f < d.fcap) { d.flag_b1[f] = b1; d.flag_tau[f] = tau; }
    }
}

// ------------------------------------------------------------------ kernel
// MODE 0: assignment of the shard (labels + near-tie flags).
// MODE 1: candidate pass over the gathered flagged rows Xf: re-computes the
//         same scores (bitwise: same operands, same MMA sequence) and emits
//         every centroid j with s_j <= b1 + tau_i -- the only centroids that
//         can be the exact argmin (refine.cu decides them in fp64).
template <int A, int MODE>   // d = 32 * A
__global__ void __launch_bounds__(TC_THREADS, 1)
k_assign_tc(const __grid_constant__ CUtensorMap tm_x, const __grid_constant__ CUtensorMap tm_chi,
            const __grid_constant__ CUtensorMap tm_clo, Dev d, GEval g, int S, int NT) {
    if (!geval_active(d, g)) return;
    long long n_rows = d.n;
    if (MODE == 1) {
        n_rows = d.flag_count[g.branch];
        if (n_rows > d.fcap) n_rows = d.fcap;
        if (n_rows == 0) return;
    }
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint8_t* xhi = smem;
    uint8_t* xlo = xhi + A * ATOM_BYTES_X;
    uint8_t* stg = xlo + A * ATOM_BYTES_X;
    float* cns = reinterpret_cast<float*>(stg + (size_t)S * STAGE_BYTES);
    uint64_t* bars = reinterpret_cast<uint64_t*>(cns + NT * TC_BN);
    uint64_t* full = bars;
    uint64_t* empty = bars + S;
    uint64_t* accf = bars + 2 * S;
    uint64_t* acce = accf + 2;
    uint64_t* xfull = acce + 2;
    uint64_t* xready = xfull + 1;
    uint64_t* xempty = xready + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(xempty + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int K = d.K;
    for (int i = threadIdx.x; i < NT * TC_BN; i += TC_THREADS) cns[i] = i < K ? d.cn[i] : INFINITY;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) { mbar_init(full + s, 1); mbar_init(empty + s, 1); }
        for (int b = 0; b < 2; ++b) { mbar_init(accf + b, 1); mbar_init(acce + b, 4); }
        mbar_init(xfull, 1); mbar_init(xready, 4); mbar_init(xempty, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_slot)),
                     "r"(2 * TC_BN));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const long long n_tiles = (n_rows + TC_BM - 1) / TC_BM;

    if (warp == 0) {
        if (lane == 0) {                                           // ---- TMA producer
            int s = 0; uint32_t ph = 0, xph = 0;
            for (long long tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
                mbar_wait(xempty, xph ^ 1);
                xph ^= 1;
                mbar_expect_tx(xfull, A * ATOM_BYTES_X);
                for (int a = 0; a < A; ++a) tma_load_2d(xhi + a * ATOM_BYTES_X, &tm_x, xfull, a * 32, (int)(tile * TC_BM));
                for (int nt = 0; nt < NT; ++nt) {
                    for (int a = 0; a < A; ++a) {
                        mbar_wait(empty + s, ph ^ 1);
                        mbar_expect_tx(full + s, STAGE_BYTES);
                        uint8_t* st = stg + (size_t)s * STAGE_BYTES;
                        tma_load_2d(st, &tm_chi, full + s, a * 32, nt * TC_BN);
                        tma_load_2d(st + TC_BN * 128, &tm_clo, full + s, a * 32, nt * TC_BN);
                        if (++s == S) { s = 0; ph ^= 1; }
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {                                           // ---- MMA issuer
            int s = 0, acc = 0; uint32_t ph = 0, xph = 0, aph = 0;
            const uint32_t xhi_a = su32(xhi), xlo_a = su32(xlo), stg_a = su32(stg);
            for (long long tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
                mbar_wait(xready, xph);
                xph ^= 1;
                tc_fence_after();
                for (int nt = 0; nt < NT; ++nt) {
                    mbar_wait(acce + acc, aph ^ 1);
                    tc_fence_after();
                    const uint32_t dt = tmem + (uint32_t)(acc * TC_BN);
                    for (int a = 0; a < A; ++a) {
                        mbar_wait(full + s, ph);
                        tc_fence_after();
                        const uint32_t sb = stg_a + (uint32_t)(s * STAGE_BYTES);
#pragma unroll
                        for (int kk = 0; kk < 4; ++kk) {
                            const uint32_t ko = (uint32_t)(kk * 32);
                            const uint64_t ah = sdesc(xhi_a + a * ATOM_BYTES_X + ko);
                            const uint64_t al = sdesc(xlo_a + a * ATOM_BYTES_X + ko);
                            const uint64_t bh = sdesc(sb + ko);
                            const uint64_t bl = sdesc(sb + TC_BN * 128 + ko);
                            mma_tf32(dt, al, bh, (a | kk) ? 1u : 0u);   // small terms first
                            mma_tf32(dt, ah, bl, 1u);
                            mma_tf32(dt, ah, bh, 1u);
                        }
                        mma_commit(empty + s);                     // frees the C stage when done
                        if (++s == S) { s = 0; ph ^= 1; }
                    }
                    mma_commit(accf + acc);                        // accumulator ready
                    if (++acc == 2) { acc = 0; aph ^= 1; }
                }
                mma_commit(xempty);                                // X tile no longer read
            }
        }
    } else if (warp >= 4) {                                        // ---- epilogue
        const int q = warp - 4;
        const int r = q * 32 + lane;                               // row in tile == TMEM lane
        int* lab_out = g.lab_out ? g.lab_out : d.lab[d.st->cur];
        const float cmax2 = __uint_as_float(d.st->cmax2_bits);
        const float gam = d.tau_gamma;
        int acc = 0; uint32_t xph = 0, aph = 0;
        for (long long tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
            // split the X tile in place: hi = tf32(x) into xhi, lo = x - hi into xlo
            mbar_wait(xfull, xph);
            xph ^= 1;
            float xn = 0.f;
#pragma unroll
            for (int a = 0; a < A; ++a) {
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    const int off = a * ATOM_BYTES_X + r * 128 + ((c ^ (r & 7)) << 4);
                    float4 v = *reinterpret_cast<float4*>(xhi + off);
                    float4 h, l;
                    h.x = __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u); l.x = v.x - h.x;
                    h.y = __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u); l.y = v.y - h.y;
                    h.z = __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u); l.z = v.z - h.z;
                    h.w = __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u); l.w = v.w - h.w;
                    xn = fmaf(v.x, v.x, xn); xn = fmaf(v.y, v.y, xn); xn = fmaf(v.z, v.z, xn); xn = fmaf(v.w, v.w, xn);
                    *reinterpret_cast<float4*>(xhi + off) = h;
                    *reinterpret_cast<float4*>(xlo + off) = l;
                }
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(xready);
            float b1 = INFINITY, b2 = INFINITY;
            int i1 = 0;
            const long long frow = tile * TC_BM + r;
            float lim = -INFINITY;
            int cnt = 0;
            if (MODE == 1 && frow < n_rows) lim = d.flag_b1[frow] + d.flag_tau[frow];
            for (int nt = 0; nt < NT; ++nt) {
                mbar_wait(accf + acc, aph);
                tc_fence_after();
                const uint32_t tbase = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * TC_BN);
#pragma unroll 1
                for (int cb = 0; cb < TC_BN / 32; ++cb) {
                    uint32_t v[32];
                    tmem_ld32(tbase + cb * 32, v);
                    const float* cnp = cns + nt * TC_BN + cb * 32;
                    const int j0 = nt * TC_BN + cb * 32;
#pragma unroll
                    for (int j = 0; j < 32; j += 4) {
                        const float4 c4 = *reinterpret_cast<const float4*>(cnp + j);
                        const float cj[4] = {c4.x, c4.y, c4.z, c4.w};
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const float sc = fmaf(-2.0f, __uint_as_float(v[j + u]), cj[u]);
                            if (MODE == 0) {
                                const bool p = sc < b1;
                                b2 = fminf(b2, fmaxf(sc, b1));
                                i1 = p ? j0 + j + u : i1;
                                b1 = fminf(b1, sc);
                            } else if (sc <= lim) {
                                if (cnt < AAKM_MAXC) d.cand[frow * AAKM_MAXC + cnt] = j0 + j + u;
                                ++cnt;
                            }
                        }
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(acce + acc);
                if (++acc == 2) { acc = 0; aph ^= 1; }
            }
            if (MODE == 0) {
                const long long row = frow;
                const bool ok = row < d.n;
                const float tau = gam * (xn + cmax2);
                if (ok) lab_out[row] = i1;
                push_flag_tc(d, g.branch, ok && (b2 - b1 <= tau), row, b1, tau);
            } else if (frow < n_rows) {
                d.cand_cnt[frow] = cnt;
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * TC_BN));
    }
}

// ------------------------------------------------------------------ host side
static int g_num_sms = 0;

static size_t smem_need(int A, int S, int NT) {
    return 1024 + (size_t)2 * A * ATOM_BYTES_X + (size_t)S * STAGE_BYTES + (size_t)NT * TC_BN * 4 + 256;
}

static int pick_stages(int A, int NT) {
    for (int S = 6; S >= 2; --S)
        if (smem_need(A, S, NT) <= (size_t)SMEM_LIMIT) return S;
    return 0;
}

bool tc_supported(int d, int K) {
    if (d % 32 != 0 || d < 32 || d > 128) return false;
    const int NT = (K + TC_BN - 1) / TC_BN;
    return pick_stages(d / 32, NT) >= 2;
}

cudaError_t setup_tc() {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    e = cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) return e;
    const void* fns[8] = {(const void*)k_assign_tc<1, 0>, (const void*)k_assign_tc<2, 0>,
                          (const void*)k_assign_tc<3, 0>, (const void*)k_assign_tc<4, 0>,
                          (const void*)k_assign_tc<1, 1>, (const void*)k_assign_tc<2, 1>,
                          (const void*)k_assign_tc<3, 1>, (const void*)k_assign_tc<4, 1>};
    for (auto f : fns) {
        e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_LIMIT);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled encoder() {
    static PFN_encodeTiled fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (PFN_encodeTiled)p;
    }
    return fn;
}

static bool encode_rows(CUtensorMap* m, const void* base, long long rows, int d, int box_rows) {
    PFN_encodeTiled enc = encoder();
    if (!enc) return false;
    cuuint64_t dims[2] = {(cuuint64_t)d, (cuuint64_t)(rows > 0 ? rows : 1)};
    cuuint64_t strides[1] = {(cuuint64_t)d * 4};
    cuuint32_t box[2] = {32, (cuuint32_t)box_rows};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// Tensor maps for one Dev (X shard + its C_hi / C_lo buffers); opaque to the runtime.
void* tc_make_maps(const Dev& d) {
    if (!tc_supported(d.d, d.K)) return nullptr;
    TcMaps* m = nullptr;
    if (posix_memalign((void**)&m, 64, sizeof(TcMaps)) != 0) return nullptr;
    bool ok = encode_rows(&m->x, d.X, d.n, d.d, TC_BM) && encode_rows(&m->chi, d.Chi, d.K, d.d, TC_BN) &&
              encode_rows(&m->clo, d.Clo, d.K, d.d, TC_BN) && encode_rows(&m->xf, d.Xf, d.fcap, d.d, TC_BM);
    if (!ok) { free(m); return nullptr; }
    return m;
}

void tc_free_maps(void* m) { free(m); }

template <int MODE>
static void launch_tc_mode(const Dev& d, const GEval& g, const TcMaps* m, cudaStream_t s) {
    const int A = d.d / 32;
    const int NT = (d.K + TC_BN - 1) / TC_BN;
    const int S = pick_stages(A, NT);
    const size_t smem = smem_need(A, S, NT);
    int grid = g_num_sms;
    const CUtensorMap& xm = MODE == 0 ? m->x : m->xf;
    if (MODE == 0) {
        const long long n_tiles = (d.n + TC_BM - 1) / TC_BM;
        if (n_tiles < grid) grid = (int)n_tiles;
    }
    if (grid < 1) grid = 1;
    switch (A) {
        case 1: k_assign_tc<1, MODE><<<grid, TC_THREADS, smem, s>>>(xm, m->chi, m->clo, d, g, S, NT); break;
        case 2: k_assign_tc<2, MODE><<<grid, TC_THREADS, smem, s>>>(xm, m->chi, m->clo, d, g, S, NT); break;
        case 3: k_assign_tc<3, MODE><<<grid, TC_THREADS, smem, s>>>(xm, m->chi, m->clo, d, g, S, NT); break;
        default: k_assign_tc<4, MODE><<<grid, TC_THREADS, smem, s>>>(xm, m->chi, m->clo, d, g, S, NT); break;
    }
}

void launch_assign_tc(const Dev& d, const GEval& g, const void* maps, cudaStream_t s) {
    launch_tc_mode<0>(d, g, static_cast<const TcMaps*>(maps), s);
}

// ---- refine for the tensor-core engine: gather -> candidate pass -> exact fp64
// one warp per flagged row, float4 lanes (d % 32 == 0 on this engine)
__global__ void __launch_bounds__(256) k_gather_flagged(Dev d, GEval g) {
    if (!geval_active(d, g)) return;
    long long nf = d.flag_count[g.branch];
    if (nf > d.fcap) nf = d.fcap;
    const int D4 = d.d >> 2;
    const int lane = threadIdx.x & 31;
    for (long long f = (long long)blockIdx.x * 8 + (threadIdx.x >> 5); f < nf; f += (long long)gridDim.x * 8) {
        const float4* src = reinterpret_cast<const float4*>(d.X + (long long)d.flag_rows[f] * d.d);
        float4* dst = reinterpret_cast<float4*>(d.Xf + f * d.d);
        for (int k = lane; k < D4; k += 32) dst[k] = __ldg(src + k);
    }
}

// Exact fp64 argmin over the candidates of each flagged row: Eq. 3 by its
// definition (direct differences); each lane owns d/32 coordinates, the warp
// reduces in a fixed xor-tree order; lowest index wins exact ties.
__global__ void __launch_bounds__(256) k_refine_exact(Dev d, GEval g) {
    if (!geval_active(d, g)) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int D = d.d;
    int* lab_out = g.lab_out ? g.lab_out : d.lab[d.st->cur];
    long long nf = d.flag_count[g.branch];
    if (nf > d.fcap) nf = d.fcap;
    for (long long f = (long long)blockIdx.x * 8 + warp; f < nf; f += (long long)gridDim.x * 8) {
        const long long row = d.flag_rows[f];
        double xv[4];
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            const int k = lane + 32 * v;
            xv[v] = k < D ? (double)__ldg(d.X + row * D + k) : 0.0;
        }
        const int cnt = d.cand_cnt[f];
        const bool all = cnt > AAKM_MAXC || cnt == 0;
        const int nc = all ? d.K : cnt;
        double bd = INFINITY;
        int bj = 0x7fffffff;
        for (int q = 0; q < nc; ++q) {
            const int j = all ? q : d.cand[f * AAKM_MAXC + q];
            double acc = 0.0;
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                const int k = lane + 32 * v;
                if (k < D) {
                    const double df = xv[v] - (double)__ldg(d.C + (long long)j * D + k);
                    acc = fma(df, df, acc);
                }
            }
#pragma unroll
            for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            if (acc < bd || (acc == bd && j < bj)) { bd = acc; bj = j; }
        }
        if (lane == 0) lab_out[row] = bj;
    }
}

void launch_refine_tc(const Dev& d, const GEval& g, const void* maps, cudaStream_t s) {
    k_gather_flagged<<<4 * g_num_sms, 256, 0, s>>>(d, g);
    launch_tc_mode<1>(d, g, static_cast<const TcMaps*>(maps), s);
    k_refine_exact<<<4 * g_num_sms, 256, 0, s>>>(d, g);
}

}  // namespace aakm
