// seed.cu -- K-Means++ seeding on the device.
//
// The paper seeds with K-Means++ among other methods (citing
// Arthur & Vassilvitskii 2007): the first center is uniform
// over the samples, every further center is drawn with probability
// proportional to D(x)^2, the squared distance to the nearest chosen center.
// This build fixes the arithmetic so the draw is exact and identical for every
// rank count (reading R-A27; the oracle's ora_seed_pp):
//   dist_i(c) = sum_k rint(((double)x_ik - (double)c_k)^2 2^t)    int64,
//               t = 50 - e, (2 max|x|)^2 < 2^e: each term < 2^50;
//   D2_i      = min over chosen centers;  M = max_i D2_i;
//   w_i       = D2_i >> sh, sh = max(0, bitlen(M) + ceil(log2 N) - 62);
//   center r  = smallest i with w_0 + ... + w_i > floor(u_r T) (T = sum w).
// Per round: k_seed_dist (one pass over X: D2 update + max; by default the pruned
// k_seed_dist_pr, which reads X only for the rows whose minimum can change), [allreduce max],
// k_seed_weights (block sums of w over contiguous row blocks), k_seed_total
// (this rank's T into its slot), [allreduce of the slots], k_seed_select (owner
// rank, block, row; the row's bits to the exchange buffer), [allreduce of the
// buffer], k_seed_commit (row -> C_out[r], index).
#include "aakm_dev.cuh"

namespace aakm {

// ---------------------------------------------------------------- helpers
__device__ __forceinline__ long long seed_term(float x, double c, double scale) {
    const double df = __dsub_rn((double)x, c);
    // rint(fl(df^2) 2^t): the scaling is exact, so one fma with 1.5 2^52 rounds
    // fl(df^2) 2^t to the nearest integer (< 2^51) exactly as the oracle's nearbyint
    const double v = __fma_rn(__dmul_rn(df, df), scale, 6755399441055744.0);
    return __double_as_longlong(v) - 0x4338000000000000LL;
}

__device__ __forceinline__ void seed_block_rows(long long n, int nb, int b, long long& r0, long long& r1) {
    const long long per = ((n + nb - 1) / nb + 15) / 16 * 16;       // multiples of 16 rows (16-B aligned D2 runs)
    r0 = min(n, (long long)b * per);
    r1 = min(n, r0 + per);
}

__device__ __forceinline__ long long warp_max_ll(long long v) {
    for (int o = 16; o; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ long long warp_sum_ll(long long v) {
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// ---------------------------------------------------------------- k_seed_dist
// D2_i = min(D2_i, dist_i(c)) for the newest center c = C_out[r] (first round:
// D2_i = dist_i(c)), and the block maxima -> atomicMax(seed_max).
// A block's rows are contiguous, so thread 0 streams them (and their D2) into a
// SEED_NS-deep shared-memory ring with 1-D bulk copies (16 KB of X per stage,
// mbarrier completion); the 8 warps read rows from shared memory: LPR = d/4
// lanes per row (float4 each), RPW = 32/LPR rows per instruction.
constexpr int SEED_STAGE = 16384;
constexpr int SEED_NS = 4;

template <int LPR> struct SeedRing {
    static constexpr int RB = 16 * LPR;
    static constexpr int TR = SEED_STAGE / RB;                        // rows per stage
    static constexpr int SLOT = SEED_STAGE + TR * 8;                  // X rows + their D2
    static constexpr int SMEM = SEED_NS * SLOT + SEED_NS * 8;
};

__device__ __forceinline__ void sd_wait(uint64_t* bar, unsigned phase) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
    unsigned done = 0;
    while (!done) {
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                     : "=r"(done) : "r"(a), "r"(phase) : "memory");
    }
}
__device__ __forceinline__ void sd_copy(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src), "r"(bytes),
                   "r"((unsigned)__cvta_generic_to_shared(bar)) : "memory");
}

template <int LPR>
__global__ void __launch_bounds__(256) k_seed_dist(Dev d, const float* c, int first, double scale, int nb) {
    if (d.st->seed_err) return;
    using SR = SeedRing<LPR>;
    constexpr int RB = SR::RB, TR = SR::TR, RPW = 32 / LPR;
    extern __shared__ __align__(128) unsigned char sm[];
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + SEED_NS * SR::SLOT);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int h = lane / LPR, c4i = lane % LPR;
    long long r0, r1;
    seed_block_rows(d.n, nb, blockIdx.x, r0, r1);
    const int nst = (int)((r1 - r0 + TR - 1) / TR);
    if (threadIdx.x == 0) {
        for (int q = 0; q < SEED_NS; ++q)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((unsigned)__cvta_generic_to_shared(full + q)) : "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    const char* Xb = reinterpret_cast<const char*>(d.X);
    auto issue = [&](int st) {                                         // thread 0 only
        const long long a = r0 + (long long)st * TR;
        const int rows = (int)min((long long)TR, r1 - a);
        unsigned char* slot = sm + (st % SEED_NS) * SR::SLOT;
        uint64_t* b = full + st % SEED_NS;
        const unsigned xb = (unsigned)(rows * RB);
        const unsigned db = first ? 0u : (unsigned)((rows * 8 + 15) & ~15);   // r0 is a multiple of 16 rows
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                     ::"r"((unsigned)__cvta_generic_to_shared(b)), "r"(xb + db) : "memory");
        sd_copy(slot, Xb + a * RB, xb, b);
        if (db) sd_copy(slot + SEED_STAGE, d.seed_d2 + a, db, b);
    };
    if (threadIdx.x == 0)
        for (int st = 0; st < min(SEED_NS, nst); ++st) issue(st);
    const float4 cf = reinterpret_cast<const float4*>(c)[c4i];
    const double c0 = cf.x, c1 = cf.y, c2 = cf.z, c3 = cf.w;
    long long mx = 0;
    for (int st = 0; st < nst; ++st) {
        const int q = st % SEED_NS;
        sd_wait(full + q, (unsigned)(st / SEED_NS) & 1u);
        const unsigned char* slot = sm + q * SR::SLOT;
        const long long* d2s = reinterpret_cast<const long long*>(slot + SEED_STAGE);
        const long long a = r0 + (long long)st * TR;
        const int rows = (int)min((long long)TR, r1 - a);
#pragma unroll 4
        for (int ib = warp * RPW; ib < TR; ib += nw * RPW) {           // uniform trip count
            const int i = ib + h;
            const bool ok = i < rows;
            const float4 x = *reinterpret_cast<const float4*>(slot + (ok ? i : 0) * RB + 16 * c4i);
            long long s = seed_term(x.x, c0, scale) + seed_term(x.y, c1, scale) +
                          seed_term(x.z, c2, scale) + seed_term(x.w, c3, scale);
#pragma unroll
            for (int o = 1; o < LPR; o <<= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            if (ok && c4i == 0) {
                const long long v = first ? s : min(s, d2s[i]);
                d.seed_d2[a + i] = v;
                mx = max(mx, v);
            }
        }
        __syncthreads();                                               // the slot is consumed
        if (threadIdx.x == 0 && st + SEED_NS < nst) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(st + SEED_NS);
        }
    }
    mx = warp_max_ll(mx);
    if (lane == 0 && mx > 0) atomicMax(reinterpret_cast<unsigned long long*>(&d.st->seed_max), (unsigned long long)mx);
}

// any d: one row per warp step, lanes over the coordinates
__global__ void __launch_bounds__(256) k_seed_dist_any(Dev d, const float* c, int first, double scale, int nb) {
    if (d.st->seed_err) return;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    long long r0, r1;
    seed_block_rows(d.n, nb, blockIdx.x, r0, r1);
    long long mx = 0;
    for (long long row = r0 + warp; row < r1; row += nw) {
        long long s = 0;
        for (int k = lane; k < d.d; k += 32) s += seed_term(__ldcs(d.X + row * d.d + k), (double)c[k], scale);
        s = warp_sum_ll(s);
        if (lane == 0) {
            const long long v = first ? s : min(s, d.seed_d2[row]);
            d.seed_d2[row] = v;
            mx = max(mx, v);
        }
    }
    mx = warp_max_ll(mx);
    if (lane == 0 && mx > 0) atomicMax(reinterpret_cast<unsigned long long*>(&d.st->seed_max), (unsigned long long)mx);
}

// ---------------------------------------------------------------- pruned D2 update
// The same D2_i = min(D2_i, dist_i(c_q)) for the newest center q, skipping every row
// whose minimum provably cannot change (triangle inequality over the chosen centers,
// as in accelerated K-Means++; the result is the same integers, so the draw is
// unchanged).  Row i keeps j = near_i with D2_i = dist_i(c_j).  In real arithmetic
//   a^2 = ||x - c_j||^2 <= (D2_i + d) 2^-t (1 + 4u)   (each term of dist is
//   rint(fl(fl(x - c)^2) 2^t): >= that square (1 - 2u)^... 2^t - 1/2),
// and if ||c_q - c_j|| >= 2 a_up (1 + 1e-9) then b = ||x - c_q|| >= a_up (1 + 2e-9), so
//   dist_i(c_q) >= b^2 2^t (1 - 4u) - d/2 >= (D2_i + d)(1 + 4e-9)(1 - 4u) - d/2 > D2_i:
// the minimum stays D2_i.  cc_j below is a lower bound of ||c_q - c_j|| (fp64, rounded
// down by a relative 1e-9, far above the few-ulp error of the d-term sum).
__global__ void __launch_bounds__(256) k_seed_cc(Dev d, const float* C, int q) {
    const int D = d.d;
    const float* cq = C + (long long)q * D;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < q; j += gridDim.x * blockDim.x) {
        const float* cj = C + (long long)j * D;
        double s = 0.0;
        for (int k = 0; k < D; ++k) {
            const double df = (double)cq[k] - (double)cj[k];
            s = fma(df, df, s);
        }
        d.seed_cc[j] = sqrt(s) * (1.0 - 1e-9);
    }
}

// Warps over 32-row batches: lane = row for the test (D2, near, cc[near]: 12 B per
// row), then the rows that need it LPR lanes per row, RPW rows per load instruction,
// U instructions in flight; the newest center is in registers (one float4 per lane).
template <int LPR>
__global__ void __launch_bounds__(256) k_seed_dist_pr(Dev d, const float* C, int q, double scale) {
    if (d.st->seed_err) return;
    constexpr int RPW = 32 / LPR, U = 4;
    __shared__ int lst[8][32];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int h = lane / LPR, c4i = lane % LPR;
    const long long wg = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const long long nwg = ((long long)gridDim.x * blockDim.x) >> 5;
    const float4 cf = reinterpret_cast<const float4*>(C + (long long)q * d.d)[c4i];
    const double c0 = cf.x, c1 = cf.y, c2 = cf.z, c3 = cf.w;
    const double two_mt = 1.0 / scale, dd = (double)d.d;            // 2^-t exact
    const float4* X4 = reinterpret_cast<const float4*>(d.X);
    long long mx = 0;
    for (long long base = wg * 32; base < d.n; base += nwg * 32) {
        const long long i = base + lane;
        const bool ok = i < d.n;
        long long D2 = 0;
        bool need = false;
        if (ok) {
            if (q == 0) {
                need = true;                                         // first center: every row
            } else {
                D2 = d.seed_d2[i];
                const int nr = d.seed_near[i];
                const double aup = sqrt(((double)D2 + dd) * two_mt * (1.0 + 1e-12)) * (1.0 + 1e-12);
                need = !(d.seed_cc[nr] >= 2.0 * aup * (1.0 + 1e-9));
                if (!need) mx = max(mx, D2);
            }
        }
        const unsigned m = __ballot_sync(0xffffffffu, need);
        const int cnt = __popc(m);
        if (need) lst[wib][__popc(m & ((1u << lane) - 1))] = lane;
        __syncwarp();
        for (int k0 = 0; k0 < cnt; k0 += U * RPW) {
            float4 xv[U];
            int src[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int k = k0 + u * RPW + h;
                src[u] = k < cnt ? lst[wib][k] : -1;
                xv[u] = src[u] >= 0 ? __ldg(X4 + (base + src[u]) * (long long)LPR + c4i) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                long long s = seed_term(xv[u].x, c0, scale) + seed_term(xv[u].y, c1, scale) +
                              seed_term(xv[u].z, c2, scale) + seed_term(xv[u].w, c3, scale);
#pragma unroll
                for (int o = 1; o < LPR; o <<= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
                const long long old = __shfl_sync(0xffffffffu, D2, src[u] >= 0 ? src[u] : 0);
                if (src[u] >= 0 && c4i == 0) {
                    const long long row = base + src[u];
                    const long long v = q == 0 ? s : min(s, old);
                    if (q == 0 || s < old) {
                        d.seed_d2[row] = v;
                        d.seed_near[row] = q;
                    }
                    mx = max(mx, v);
                }
            }
        }
        __syncwarp();
    }
    mx = warp_max_ll(mx);
    if (lane == 0 && mx > 0) atomicMax(reinterpret_cast<unsigned long long*>(&d.st->seed_max), (unsigned long long)mx);
}

__device__ __forceinline__ int seed_shift(const Dev& d, int log2n) {
    const unsigned long long M = d.st->seed_max;
    const int bl = M ? 64 - __clzll((long long)M) : 0;
    return max(0, bl + log2n - 62);
}

// ---------------------------------------------------------------- k_seed_weights
// part[b] = sum of w_i over block b's rows (the same contiguous blocks).
__global__ void __launch_bounds__(256) k_seed_weights(Dev d, int log2n, int nb) {
    if (d.st->seed_err) return;
    __shared__ long long ws[8];
    const int sh = seed_shift(d, log2n);
    long long r0, r1;
    seed_block_rows(d.n, nb, blockIdx.x, r0, r1);
    long long s = 0;
    for (long long i = r0 + threadIdx.x; i < r1; i += blockDim.x) s += d.seed_d2[i] >> sh;
    s = warp_sum_ll(s);
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        long long t = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += ws[w];
        d.seed_part[blockIdx.x] = t;
    }
}

// ---------------------------------------------------------------- block scan helper
// Inclusive scan of one int64 per thread over a 1024-thread block; returns the
// inclusive prefix, total in *tot.
__device__ long long block_scan_incl(long long v, long long* sm32, long long* tot) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int o = 1; o < 32; o <<= 1) {
        const long long t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += t;
    }
    if (lane == 31) sm32[w] = v;
    __syncthreads();
    if (w == 0) {
        long long x = lane < (int)(blockDim.x >> 5) ? sm32[lane] : 0;
        for (int o = 1; o < 32; o <<= 1) {
            const long long t = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += t;
        }
        sm32[lane] = x;
    }
    __syncthreads();
    const long long r = v + (w ? sm32[w - 1] : 0);
    *tot = sm32[(blockDim.x >> 5) - 1];
    __syncthreads();
    return r;
}

// ---------------------------------------------------------------- k_seed_total
// this rank's T into seed_T[rank] (the other slots zero: a sum-allreduce of the
// slots is an allgather); an all-zero M is the "fewer than k distinct" error.
__global__ void __launch_bounds__(1024) k_seed_total(Dev d, int nb, int rank, int nranks) {
    __shared__ long long sm32[32];
    long long v = 0;
    for (int b = threadIdx.x; b < nb; b += blockDim.x) v += d.seed_part[b];
    long long tot;
    block_scan_incl(v, sm32, &tot);
    if (threadIdx.x < nranks) d.seed_T[threadIdx.x] = threadIdx.x == rank ? tot : 0;
}

// ---------------------------------------------------------------- k_seed_select
// Global T and tau = min(T - 1, floor(u T)); the owner rank walks its blocks and
// then its rows; the chosen row's bits and global index go to seed_x (zeros on
// the other ranks, so a sum-allreduce delivers them everywhere).
__global__ void __launch_bounds__(1024) k_seed_select(Dev d, int r, int log2n, int nb, int rank, int nranks,
                                                      long long row_offset) {
    __shared__ long long sm32[32];
    __shared__ long long s_tau, s_base;
    __shared__ int s_blk, s_owner;
    int* xo = d.seed_x;
    const int D = d.d;
    for (int k = threadIdx.x; k < D + 2; k += blockDim.x) xo[k] = 0;
    if (d.st->seed_err) return;
    if (d.st->seed_max == 0) {                      // every sample sits on a chosen center
        if (threadIdx.x == 0) d.st->seed_err = 2;
        return;
    }
    if (threadIdx.x == 0) {
        long long T = 0;
        for (int q = 0; q < nranks; ++q) T += d.seed_T[q];
        long long tau = (long long)floor(d.seed_u[r] * (double)T);
        if (tau > T - 1) tau = T - 1;
        int owner = 0;
        long long acc = 0;
        for (; owner < nranks; ++owner) {               // first rank whose cumulative total passes tau
            if (acc + d.seed_T[owner] > tau) break;
            acc += d.seed_T[owner];
        }
        s_owner = owner;
        s_tau = tau - acc;                              // within the owner's rows
    }
    __syncthreads();
    if (s_owner != rank) return;
    const int sh = seed_shift(d, log2n);
    const long long tau = s_tau;
    // block: first b with part[0] + ... + part[b] > tau (nb <= 2 per thread)
    {
        const int per = (nb + blockDim.x - 1) / blockDim.x;
        const int b0 = threadIdx.x * per;
        long long v = 0;
        for (int b = b0; b < min(nb, b0 + per); ++b) v += d.seed_part[b];
        long long tot;
        const long long incl = block_scan_incl(v, sm32, &tot);
        const long long excl = incl - v;
        if (excl <= tau && tau < incl) {
            long long a = excl;
            for (int b = b0; b < min(nb, b0 + per); ++b) {
                if (a + d.seed_part[b] > tau) { s_blk = b; s_base = a; break; }
                a += d.seed_part[b];
            }
        }
        __syncthreads();
    }
    // row within block s_blk: contiguous row chunks per thread, then one walk
    long long r0, r1;
    seed_block_rows(d.n, nb, s_blk, r0, r1);
    const long long tl = tau - s_base;
    const long long per = (r1 - r0 + blockDim.x - 1) / blockDim.x;
    const long long q0 = r0 + threadIdx.x * per, q1 = min(r1, q0 + per);
    long long v = 0;
    for (long long i = q0; i < q1; ++i) v += d.seed_d2[i] >> sh;
    long long tot;
    const long long incl = block_scan_incl(v, sm32, &tot);
    const long long excl = incl - v;
    if (excl <= tl && tl < incl) {
        long long a = excl;
        for (long long i = q0; i < q1; ++i) {
            a += d.seed_d2[i] >> sh;
            if (a > tl) {
                const float* x = d.X + i * D;
                for (int k = 0; k < D; ++k) xo[k] = __float_as_int(x[k]);
                const long long gi = row_offset + i;
                xo[D] = (int)(gi & 0xffffffffLL);
                xo[D + 1] = (int)(gi >> 32);
                break;
            }
        }
    }
}

// first center: the owner of global row i0 writes it (row_local >= 0 on the owner only)
__global__ void k_seed_first(Dev d, long long row_local, long long gi) {
    int* xo = d.seed_x;
    const int D = d.d;
    for (int k = threadIdx.x; k < D + 2; k += blockDim.x) {
        int v = 0;
        if (row_local >= 0) v = k < D ? __float_as_int(d.X[row_local * D + k]) : (k == D ? (int)(gi & 0xffffffffLL) : (int)(gi >> 32));
        xo[k] = v;
    }
}

// seed_x -> C_out[r], seed_idx[r]; resets the max for the next round
__global__ void k_seed_commit(Dev d, float* C_out, int r) {
    const int D = d.d;
    const int* xo = d.seed_x;
    for (int k = threadIdx.x; k < D; k += blockDim.x) C_out[(long long)r * D + k] = __int_as_float(xo[k]);
    if (threadIdx.x == 0) {
        d.seed_idx[r] = (long long)(unsigned)xo[D] | ((long long)xo[D + 1] << 32);
        d.st->seed_max = 0;
    }
}

// ---------------------------------------------------------------- launchers
template <int LPR> static cudaError_t seed_attr() {
    return cudaFuncSetAttribute(k_seed_dist<LPR>, cudaFuncAttributeMaxDynamicSharedMemorySize, SeedRing<LPR>::SMEM);
}
cudaError_t setup_seed() {
    for (cudaError_t e : {seed_attr<1>(), seed_attr<2>(), seed_attr<4>(), seed_attr<8>(), seed_attr<16>(), seed_attr<32>()})
        if (e != cudaSuccess) return e;
    return cudaSuccess;
}

int seed_blocks(const Dev& d) {
    long long nb = (d.n + 4095) / 4096;
    if (nb > AAKM_SEED_BLOCKS) nb = AAKM_SEED_BLOCKS;
    return (int)(nb < 1 ? 1 : nb);
}

void launch_seed_first(const Dev& d, long long row_local, long long gi, cudaStream_t s) {
    k_seed_first<<<1, 128, 0, s>>>(d, row_local, gi);
}

// AAKM_SEED_PRUNE=0: every round streams all of X (k_seed_dist); default: the pruned
// update (k_seed_dist_pr, same integers) for d % 4 == 0 with d / 4 a power of two <= 32
static bool seed_prune() {
    static const bool v = !(getenv("AAKM_SEED_PRUNE") && atoi(getenv("AAKM_SEED_PRUNE")) == 0);
    return v;
}

int launch_seed_dist(const Dev& d, const float* C, int q, double scale, cudaStream_t s) {
    const int nb = seed_blocks(d);
    const int lpr = d.d / 4;
    const float* c = C + (long long)q * d.d;
    const int first = q == 0;
    if (d.d % 4 == 0 && lpr <= 32 && (lpr & (lpr - 1)) == 0 && seed_prune() && ((uintptr_t)d.X & 15) == 0) {
        if (q > 0) k_seed_cc<<<(q + 255) / 256, 256, 0, s>>>(d, C, q);
        const int nl = q > 0 ? 2 : 1;
        const int pb = 8 * d.num_sms;
        switch (lpr) {
            case 1: k_seed_dist_pr<1><<<pb, 256, 0, s>>>(d, C, q, scale); return nl;
            case 2: k_seed_dist_pr<2><<<pb, 256, 0, s>>>(d, C, q, scale); return nl;
            case 4: k_seed_dist_pr<4><<<pb, 256, 0, s>>>(d, C, q, scale); return nl;
            case 8: k_seed_dist_pr<8><<<pb, 256, 0, s>>>(d, C, q, scale); return nl;
            case 16: k_seed_dist_pr<16><<<pb, 256, 0, s>>>(d, C, q, scale); return nl;
            default: k_seed_dist_pr<32><<<pb, 256, 0, s>>>(d, C, q, scale); return nl;
        }
    }
    if (d.d % 4 == 0 && lpr <= 32 && (lpr & (lpr - 1)) == 0) {
        switch (lpr) {
            case 1: k_seed_dist<1><<<nb, 256, SeedRing<1>::SMEM, s>>>(d, c, first, scale, nb); return 1;
            case 2: k_seed_dist<2><<<nb, 256, SeedRing<2>::SMEM, s>>>(d, c, first, scale, nb); return 1;
            case 4: k_seed_dist<4><<<nb, 256, SeedRing<4>::SMEM, s>>>(d, c, first, scale, nb); return 1;
            case 8: k_seed_dist<8><<<nb, 256, SeedRing<8>::SMEM, s>>>(d, c, first, scale, nb); return 1;
            case 16: k_seed_dist<16><<<nb, 256, SeedRing<16>::SMEM, s>>>(d, c, first, scale, nb); return 1;
            default: k_seed_dist<32><<<nb, 256, SeedRing<32>::SMEM, s>>>(d, c, first, scale, nb); return 1;
        }
    }
    k_seed_dist_any<<<nb, 256, 0, s>>>(d, c, first, scale, nb);
    return 1;
}

void launch_seed_weights(const Dev& d, int log2n, int rank, int nranks, cudaStream_t s) {
    const int nb = seed_blocks(d);
    k_seed_weights<<<nb, 256, 0, s>>>(d, log2n, nb);
    k_seed_total<<<1, 1024, 0, s>>>(d, nb, rank, nranks);
}

void launch_seed_select(const Dev& d, int r, int log2n, int rank, int nranks, long long row_offset, cudaStream_t s) {
    k_seed_select<<<1, 1024, 0, s>>>(d, r, log2n, seed_blocks(d), rank, nranks, row_offset);
}

void launch_seed_commit(const Dev& d, float* C_out, int r, cudaStream_t s) {
    k_seed_commit<<<1, 128, 0, s>>>(d, C_out, r);
}

}  // namespace aakm
