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

// ------------------------------------------------------------------
// Sorted engine for large shards (n >= AAKM_SORTED_MIN_ROWS): rows are
// bucketed by label, then each warp sums a chunk of <= SEG_ROWS rows of one
// cluster in fp64 registers (lanes over d) and issues d atomics per chunk
// instead of d per row.  X is read exactly once, as contiguous row segments;
// the energy uses the chunk's centroid kept in registers.
//   k_hist     N_j (block histograms in smem) + #changed + label check
//   k_scan     offsets, per-cluster chunk counts, cursors, N_j -> packed
//   k_scatter  perm[offset_j + rank] = row (warp-aggregated cursors)
//   k_segsum   S_j += sum of the chunk's rows, E += sum (x - c_j)^2

constexpr int SEG_ROWS = 256;

__device__ __forceinline__ void finish_changed(const Dev& d, double* out, long long ch) {
    __shared__ long long sc[32];
    __shared__ bool last;
    for (int o = 16; o; o >>= 1) ch += __shfl_xor_sync(0xffffffffu, ch, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
    if (l == 0) sc[w] = ch;
    __syncthreads();
    if (threadIdx.x == 0) {
        long long bc = 0;
        for (int i = 0; i < nw; ++i) bc += sc[i];
        d.upd_part[2 * blockIdx.x + 1] = __longlong_as_double(bc);
        __threadfence();
        last = atomicAdd(&d.st->hist_ctr, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    long long tc = 0;
    for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x)
        tc += __double_as_longlong(__ldcg(d.upd_part + 2 * b + 1));
    for (int o = 16; o; o >>= 1) tc += __shfl_xor_sync(0xffffffffu, tc, o);
    __syncthreads();
    if (l == 0) sc[w] = tc;
    __syncthreads();
    if (threadIdx.x == 0) {
        long long bc = 0;
        for (int i = 0; i < nw; ++i) bc += sc[i];
        out[(long long)d.K * d.d + d.K + 1] += (double)bc;
        d.st->hist_ctr = 0;
    }
}

__global__ void __launch_bounds__(256) k_hist(Dev d, GEval g) {
    if (!geval_active(d, g)) return;
    const Pick p = pick(d, g);
    extern __shared__ int hs[];
    const int K = d.K;
    const bool use_smem = K <= 16384;
    if (use_smem) {
        for (int j = threadIdx.x; j < K; j += blockDim.x) hs[j] = 0;
        __syncthreads();
    }
    long long ch = 0;
    int bad = 0;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < d.n;
         i += (long long)gridDim.x * blockDim.x) {
        const int j = p.lab[i];
        if (j < 0 || j >= K) { bad = 1; continue; }
        if (p.prev) ch += (p.prev[i] != j);
        if (use_smem) atomicAdd(&hs[j], 1);
        else atomicAdd(&d.seg_count[j], 1);
    }
    if (bad) d.st->label_error = 1;
    if (use_smem) {
        __syncthreads();
        for (int j = threadIdx.x; j < K; j += blockDim.x)
            if (hs[j]) atomicAdd(&d.seg_count[j], hs[j]);
    }
    finish_changed(d, p.out, ch);
}

// one block: exclusive scans over K (counts -> offsets, chunks -> chunk offsets)
__global__ void __launch_bounds__(1024) k_scan(Dev d, GEval g) {
    if (!geval_active(d, g)) return;
    const Pick p = pick(d, g);
    const int K = d.K;
    const long long KD = (long long)K * d.d;
    __shared__ long long wsum[2][32];
    __shared__ long long carry[2];
    if (threadIdx.x == 0) { carry[0] = 0; carry[1] = 0; }
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int base = 0; base < K; base += blockDim.x) {
        const int j = base + threadIdx.x;
        const long long c = j < K ? d.seg_count[j] : 0;
        const long long nc = (c + SEG_ROWS - 1) / SEG_ROWS;
        long long a = c, b = nc;
        for (int o = 1; o < 32; o <<= 1) {
            const long long ta = __shfl_up_sync(0xffffffffu, a, o), tb = __shfl_up_sync(0xffffffffu, b, o);
            if (lane >= o) { a += ta; b += tb; }
        }
        if (lane == 31) { wsum[0][w] = a; wsum[1][w] = b; }
        __syncthreads();
        if (w == 0) {
            long long x = lane < (int)(blockDim.x >> 5) ? wsum[0][lane] : 0;
            long long y = lane < (int)(blockDim.x >> 5) ? wsum[1][lane] : 0;
            for (int o = 1; o < 32; o <<= 1) {
                const long long tx = __shfl_up_sync(0xffffffffu, x, o), ty = __shfl_up_sync(0xffffffffu, y, o);
                if (lane >= o) { x += tx; y += ty; }
            }
            wsum[0][lane] = x; wsum[1][lane] = y;
        }
        __syncthreads();
        const long long pa = (w ? wsum[0][w - 1] : 0) + a - c + carry[0];
        const long long pb = (w ? wsum[1][w - 1] : 0) + b - nc + carry[1];
        if (j < K) {
            d.seg_off[j] = (int)pa;
            d.seg_cursor[j] = (int)pa;
            d.seg_chunk[j] = (int)pb;
            p.out[KD + j] = (double)c;                  // N_j
        }
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) { carry[0] = pa + c; carry[1] = pb + nc; }
        __syncthreads();
    }
    if (threadIdx.x == 0) { d.seg_off[K] = (int)carry[0]; d.seg_chunk[K] = (int)carry[1]; }
}

__global__ void __launch_bounds__(256) k_scatter(Dev d, GEval g) {
    if (!geval_active(d, g)) return;
    const Pick p = pick(d, g);
    const int K = d.K;
    const int lane = threadIdx.x & 31;
    for (long long i0 = (long long)blockIdx.x * blockDim.x; i0 < d.n; i0 += (long long)gridDim.x * blockDim.x) {
        const long long i = i0 + threadIdx.x;
        int j = i < d.n ? p.lab[i] : -1;
        if (j >= K) j = -1;
        const unsigned peers = __match_any_sync(0xffffffffu, j);
        const int leader = __ffs(peers) - 1;
        int base = 0;
        if (lane == leader && j >= 0) base = atomicAdd(&d.seg_cursor[j], __popc(peers));
        base = __shfl_sync(peers, base, leader);
        if (j >= 0) d.perm[base + __popc(peers & ((1u << lane) - 1))] = (int)i;
    }
}

template <int V>   // floats per lane: d <= 32 * V
__global__ void __launch_bounds__(256) k_segsum(Dev d, GEval g) {
    if (!geval_active(d, g)) return;
    const Pick p = pick(d, g);
    const int D = d.d, K = d.K;
    const int lane = threadIdx.x & 31;
    const long long nchunks = d.seg_chunk[K];
    double e_acc = 0.0;
    for (long long w = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); w < nchunks;
         w += (long long)gridDim.x * (blockDim.x >> 5)) {
        // cluster of chunk w: last j with seg_chunk[j] <= w
        int lo = 0, hi = K - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (d.seg_chunk[mid] <= w) lo = mid; else hi = mid - 1;
        }
        const int j = lo;
        const long long r0 = d.seg_off[j] + (w - d.seg_chunk[j]) * SEG_ROWS;
        const long long r1 = min((long long)d.seg_off[j + 1], r0 + SEG_ROWS);
        float c[V];
        double s[V];
#pragma unroll
        for (int v = 0; v < V; ++v) {
            const int k = lane + 32 * v;
            c[v] = k < D ? __ldg(p.C + (long long)j * D + k) : 0.f;
            s[v] = 0.0;
        }
        long long q = r0;
        for (; q + 4 <= r1; q += 4) {
            int rows[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) rows[u] = d.perm[q + u];
            float xv[4][V];
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int v = 0; v < V; ++v) {
                    const int k = lane + 32 * v;
                    xv[u][v] = k < D ? __ldcs(d.X + (long long)rows[u] * D + k) : 0.f;
                }
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int v = 0; v < V; ++v) {
                    s[v] += (double)xv[u][v];
                    const double df = (double)xv[u][v] - (double)c[v];
                    e_acc = fma(df, df, e_acc);
                }
        }
        for (; q < r1; ++q) {
            const int row = d.perm[q];
#pragma unroll
            for (int v = 0; v < V; ++v) {
                const int k = lane + 32 * v;
                const float x = k < D ? __ldcs(d.X + (long long)row * D + k) : 0.f;
                s[v] += (double)x;
                const double df = (double)x - (double)c[v];
                e_acc = fma(df, df, e_acc);
            }
        }
#pragma unroll
        for (int v = 0; v < V; ++v) {
            const int k = lane + 32 * v;
            if (k < D) red_add_f64(p.out + (long long)j * D + k, s[v]);
        }
    }
    finish_scalars(d, p.out, e_acc, 0);
}

cudaError_t setup_update() { return cudaFuncSetAttribute(k_hist, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536); }

bool update_sorted(const Dev& d) { return d.n >= AAKM_SORTED_MIN_ROWS && d.d <= 128; }

void launch_update(const Dev& d, const GEval& g, cudaStream_t s) {
    if (!update_sorted(d)) {
        k_update<<<d.upd_blocks, 256, 0, s>>>(d, g);
        return;
    }
    cudaMemsetAsync(d.seg_count, 0, (size_t)d.K * 4, s);
    const size_t hs = d.K <= 16384 ? (size_t)d.K * 4 : 0;
    k_hist<<<d.upd_blocks, 256, hs, s>>>(d, g);
    k_scan<<<1, 1024, 0, s>>>(d, g);
    k_scatter<<<d.upd_blocks, 256, 0, s>>>(d, g);
    const int V = (d.d + 31) / 32;
    switch (V) {
        case 1: k_segsum<1><<<d.upd_blocks, 256, 0, s>>>(d, g); break;
        case 2: k_segsum<2><<<d.upd_blocks, 256, 0, s>>>(d, g); break;
        case 3: k_segsum<3><<<d.upd_blocks, 256, 0, s>>>(d, g); break;
        default: k_segsum<4><<<d.upd_blocks, 256, 0, s>>>(d, g); break;
    }
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
