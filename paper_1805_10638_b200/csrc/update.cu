// update.cu -- update step partials + exact energy + convergence count.
//
// Update step, Eq. (4): c_j = (1/N_j) sum_{rho_i = j} x_i.
// One pass over the local shard produces the packed vector that the ranks
// allreduce:
//   S_j  = sum_{rho_i = j} x_i           (fp64; the mean is G_j = S_j / N_j)
//   N_j  = #{i : rho_i = j}
//   E    = sum_i ||x_i - c_{rho_i}||^2  (Eq. 1 with the given P, PAPER.md:113;
//                                         fp64 direct differences)
//   changed = #{i : rho_i != rho_i^{prev}}
// The energy reuses the same loads of x_i and c_{rho_i}, so X is read once.
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

// Lanes are grouped per row (group = next pow2 >= d, <= 32) so a row's d
// coordinates are read and reduced as one coalesced segment; S_j and N_j go
// to global memory with fp64 red.global.add (native on sm_100a; the fp32
// shared-memory atomics compile to CAS loops and measured slower).
__global__ void __launch_bounds__(256) k_update(Dev d, GEval g) {
    if (!geval_active(d, g)) return;
    const Pick p = pick(d, g);
    const int D = d.d, K = d.K;
    const long long KD = (long long)K * D;
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
            red_add_f64(p.out + KD + j, 1.0);
        }
        const float* x = d.X + row * D;
        const float* c = p.C + (long long)j * D;
        for (int k = gl; k < D; k += GS) {
            const float xv = __ldcs(x + k);
            const double diff = (double)xv - (double)__ldg(c + k);   // exact in fp64
            e_acc = fma(diff, diff, e_acc);
            red_add_f64(p.out + (long long)j * D + k, (double)xv);
        }
    }
    if (bad) d.st->label_error = 1;
    finish_scalars(d, p.out, e_acc, ch);
}

cudaError_t setup_update() { return cudaSuccess; }

void launch_update(const Dev& d, const GEval& g, cudaStream_t s) {
    k_update<<<d.upd_blocks, 256, 0, s>>>(d, g);
}

// kmeans_update API: G = S / N (empty -> C_prev row, R-A15), counts.
__global__ void k_update_G(long long KD, int D, int K, const double* packed, const float* Cprev,
                           float* G, long long* counts) {
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < KD;
         e += (long long)gridDim.x * blockDim.x) {
        const int j = (int)(e / D);
        const double nj = packed[KD + j];
        G[e] = nj > 0.0 ? (float)(packed[e] / nj) : Cprev[e];
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
