// update.cu -- update step partials + exact energy + convergence count.
//
// Update step, Eq. (4): c_j = (1/N_j) sum_{rho_i = j} x_i.
// One pass over the local shard produces the packed vector that the ranks
// allreduce:
//   S'_j = sum_{rho_i = j} (x_i - c_j)   (centred on the centroids C the
//                                         assignment was made against; the
//                                         mean is G_j = c_j + S'_j / N_j)
//   N_j  = #{i : rho_i = j}
//   E    = sum_i ||x_i - c_{rho_i}||^2  (Eq. 1 with the given P, PAPER.md:113;
//                                         fp64 direct differences)
//   changed = #{i : rho_i != rho_i^{prev}}
// Centring keeps the fp32 shared-memory partial sums small (accuracy), the
// energy reuses the same loads of x_i and c_{rho_i}, so X is read once.
//
// Two engines:
//  * smem (K*d small): lanes grouped per row (group = next pow2 >= d, <= 32),
//    shared-memory privatised fp32 S' and int N, flushed once per block with
//    global fp64 atomics (red.global.add.f64);
//  * global (large K*d): same mapping, fp64 atomics straight to the packed
//    vector (coalesced: a row's d doubles are contiguous).
// E/changed: fixed-order per-block partials, reduced by the last block in a
// fixed tree -> bitwise reproducible for a fixed launch geometry.
#include "aakm_dev.cuh"

namespace aakm {

__device__ __forceinline__ void red_add_f64(double* p, double v) {
    asm volatile("red.global.add.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}

struct Pick {
    const int* lab;
    const int* prev;
    const float* C;
    double* out;
};

__device__ __forceinline__ Pick pick(const Dev& d, const GEval& g) {
    Pick p;
    const int cur = d.st->cur;
    p.lab = g.lab_out ? g.lab_out : d.lab[cur];
    p.prev = g.prev_mode == 0 ? d.lab[cur ^ 1] : (g.prev_mode == 2 ? g.lab_prev : nullptr);
    p.C = g.Cassign ? g.Cassign : d.C;
    p.out = g.packed_out ? g.packed_out : d.packed[g.branch];
    return p;
}

// Block reduction of (E, changed) and the deterministic last-block finish.
__device__ void finish_scalars(const Dev& d, double* out, double e, long long ch) {
    __shared__ double se[32];
    __shared__ long long sc[32];
    __shared__ bool last;
    for (int o = 16; o; o >>= 1) {
        e += __shfl_xor_sync(0xffffffffu, e, o);
        ch += __shfl_xor_sync(0xffffffffu, ch, o);
    }
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
    if (l == 0) { se[w] = e; sc[w] = ch; }
    __syncthreads();
    if (threadIdx.x == 0) {
        double be = 0.0; long long bc = 0;
        for (int i = 0; i < nw; ++i) { be += se[i]; bc += sc[i]; }
        d.upd_part[2 * blockIdx.x] = be;
        d.upd_part[2 * blockIdx.x + 1] = __longlong_as_double(bc);
        __threadfence();
        unsigned prevc = atomicAdd(&d.st->upd_ctr, 1u);
        last = (prevc == gridDim.x - 1);
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    double te = 0.0; long long tc = 0;
    for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) {
        te += __ldcg(d.upd_part + 2 * b);
        tc += __double_as_longlong(__ldcg(d.upd_part + 2 * b + 1));
    }
    for (int o = 16; o; o >>= 1) {
        te += __shfl_xor_sync(0xffffffffu, te, o);
        tc += __shfl_xor_sync(0xffffffffu, tc, o);
    }
    __syncthreads();
    if (l == 0) { se[w] = te; sc[w] = tc; }
    __syncthreads();
    if (threadIdx.x == 0) {
        double be = 0.0; long long bc = 0;
        for (int i = 0; i < nw; ++i) { be += se[i]; bc += sc[i]; }
        const long long KD = (long long)d.K * d.d;
        out[KD + d.K] += be;            // packed was zeroed before the launch
        out[KD + d.K + 1] += (double)bc;
        d.st->upd_ctr = 0;
    }
}

template <bool SMEM>
__global__ void __launch_bounds__(256) k_update(Dev d, GEval g) {
    if (!geval_active(d, g)) return;
    const Pick p = pick(d, g);
    const int D = d.d, K = d.K;
    const long long KD = (long long)K * D;
    extern __shared__ float4 smem4[];
    float* Ss = reinterpret_cast<float*>(smem4);       // K*D (SMEM only)
    float* Cs = Ss + KD;                               // K*D
    int* Ns = reinterpret_cast<int*>(Cs + KD);         // K
    if (SMEM) {
        for (long long e = threadIdx.x; e < KD; e += blockDim.x) { Ss[e] = 0.f; Cs[e] = p.C[e]; }
        for (int e = threadIdx.x; e < K; e += blockDim.x) Ns[e] = 0;
        __syncthreads();
    }
    int GS = 1;
    while (GS < D && GS < 32) GS <<= 1;
    const int lane = threadIdx.x & 31;
    const int gl = lane % GS;                     // lane within the row group
    const int groups_per_block = blockDim.x / GS;
    const long long gid = (long long)blockIdx.x * groups_per_block + threadIdx.x / GS;
    const long long ngroups = (long long)gridDim.x * groups_per_block;
    double e_acc = 0.0;
    long long ch = 0;
    int bad = 0;
    for (long long row = gid; row < d.n; row += ngroups) {
        const int j = p.lab[row];
        if (j < 0 || j >= K) { bad = 1; continue; }
        if (gl == 0) {
            if (p.prev) ch += (p.prev[row] != j);
            if (SMEM) atomicAdd(&Ns[j], 1);
            else red_add_f64(p.out + KD + j, 1.0);
        }
        const float* x = d.X + row * D;
        for (int k = gl; k < D; k += GS) {
            const float xv = __ldcs(x + k);
            const float cv = SMEM ? Cs[(long long)j * D + k] : __ldg(p.C + (long long)j * D + k);
            const double diff = (double)xv - (double)cv;   // exact in fp64
            e_acc = fma(diff, diff, e_acc);
            if (SMEM) atomicAdd(&Ss[(long long)j * D + k], xv - cv);
            else red_add_f64(p.out + (long long)j * D + k, diff);
        }
    }
    if (bad) d.st->label_error = 1;
    if (SMEM) {
        __syncthreads();
        for (long long e = threadIdx.x; e < KD; e += blockDim.x)
            if (Ss[e] != 0.f) red_add_f64(p.out + e, (double)Ss[e]);
        for (int e = threadIdx.x; e < K; e += blockDim.x)
            if (Ns[e]) red_add_f64(p.out + KD + e, (double)Ns[e]);
    }
    finish_scalars(d, p.out, e_acc, ch);
}

static size_t smem_bytes(const Dev& d) { return (size_t)d.K * d.d * 8 + (size_t)d.K * 4; }

cudaError_t setup_update() {
    return cudaFuncSetAttribute(k_update<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
}

void launch_update(const Dev& d, const GEval& g, cudaStream_t s) {
    const size_t sm = smem_bytes(d);
    if (sm <= 160 * 1024) {
        k_update<true><<<d.upd_blocks, 256, sm, s>>>(d, g);
    } else {
        k_update<false><<<d.upd_blocks, 256, 0, s>>>(d, g);
    }
}

// kmeans_update API: G = C_prev + S'/N (empty -> C_prev row), counts.
__global__ void k_update_G(long long KD, int D, int K, const double* packed, const float* Cprev,
                           float* G, long long* counts) {
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < KD;
         e += (long long)gridDim.x * blockDim.x) {
        const int j = (int)(e / D);
        const double nj = packed[KD + j];
        G[e] = nj > 0.0 ? (float)((double)Cprev[e] + packed[e] / nj) : Cprev[e];
        if (counts && e % D == 0) counts[j] = (long long)nj;
    }
}

void launch_update_G(const Dev& d, const double* packed, const float* Cprev, float* G,
                     long long* counts, cudaStream_t s) {
    long long KD = (long long)d.K * d.d;
    int blocks = (int)((KD + 255) / 256);
    if (blocks > 1184) blocks = 1184;
    k_update_G<<<blocks, 256, 0, s>>>(KD, d.d, d.K, packed, Cprev, G, counts);
}

}  // namespace aakm
