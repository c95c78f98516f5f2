// update.cu -- update step partials + convergence count.
//
// Update step, Eq. (4): c_j = (1/N_j) sum_{rho_i = j} x_i.
// One pass over the local shard produces the packed int64 vector the ranks
// allreduce:
//   S_j  = sum_{rho_i = j} x_i  as two fixed-point integers per coordinate:
//          x 2^(22-e) = hi + lo 2^-22 (|x| <= 2^e over all ranks, hi/lo rounded
//          to nearest), so every x with |x| >= 2^(e-23) is carried exactly and
//          the rest to 2^(e-45); integer sums are exact and order-free, so S
//          (and everything downstream) is bitwise identical run to run and for
//          any number of ranks
//   N_j  = #{i : rho_i = j}
//   E    = sum_i ||x_i - c_{rho_i}||^2  (Eq. 1 with the given P):
//          each row by direct differences in fp64 (fixed order), then the same
//          kind of two-part fixed point (energy_q): exact zeros stay zero
//   changed = #{i : rho_i != rho_i^{prev}}
// X is read once.
#include "aakm_dev.cuh"

namespace aakm {

__device__ __forceinline__ void red_add_f64(double* p, double v) {
    asm volatile("red.global.add.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}

struct Pick {
    const int* lab;
    const int* prev;
    const float* C;
    long long* out;       // packed [S_hi | S_lo | N | E | changed]
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

// x -> (hi, lo) with x 2^(22-e) = hi + lo 2^-22 (+ |residual| <= 2^-23), both
// rounded to nearest through the 1.5 * 2^23 magic (fp32 only; |x 2^(22-e)| <= 2^22).
__device__ __forceinline__ void fx_add(float x, float sc, int& hi, int& lo) {
    const float M = 12582912.0f;
    const float t = fmaf(x, sc, M);
    const float hv = t - M;
    const float r = fmaf(x, sc, -hv);                 // exact
    const float t2 = fmaf(r, 4194304.0f, M);
    hi += __float_as_int(t) - 0x4B400000;
    lo += __float_as_int(t2) - 0x4B400000;
}
__device__ __forceinline__ void red_add_s64(long long* p, long long v) {
    atomicAdd(reinterpret_cast<unsigned long long*>(p), (unsigned long long)v);
}

__device__ void finish_changed(const Dev& d, long long* out, long long ch);

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
    const int gpw = 32 / GS;                      // row groups per warp
    // warp-uniform trip count (the energy shuffles need the whole warp)
    const long long wid = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    const float sc = d.fx_scale;
    const double q = energy_q(d);
    long long ch = 0, ehi = 0, elo = 0;
    int bad = 0;
    for (long long base = wid * gpw; base < d.n; base += nw * gpw) {
        const long long row = base + lane / GS;
        const bool live = row < d.n;
        const int j = live ? p.lab[row] : 0;
        const bool okj = live && j >= 0 && j < K;   // uniform within the row group
        if (live && !okj) bad = 1;
        double e = 0.0;
        if (okj) {
            if (gl == 0) {
                if (p.prev) ch += (p.prev[row] != j);
                red_add_s64(p.out + pk_n(d) + j, 1);
            }
            const float* x = d.X + row * D;
            const float* c = p.C + (long long)j * D;
            for (int k = gl; k < D; k += GS) {
                const float xv = __ldcs(x + k);
                int hi = 0, lo = 0;
                fx_add(xv, sc, hi, lo);
                red_add_s64(p.out + (long long)j * D + k, hi);
                red_add_s64(p.out + KD + (long long)j * D + k, lo);
                const double df = (double)xv - (double)__ldg(c + k);
                e = fma(df, df, e);
            }
        }
        for (int o = 1; o < GS; o <<= 1) e += __shfl_xor_sync(0xffffffffu, e, o);   // fixed tree
        if (okj && gl == 0) energy_add(e, q, ehi, elo);
    }
    if (bad) d.st->label_error = 1;
    for (int o = 16; o; o >>= 1) {
        ehi += __shfl_xor_sync(0xffffffffu, ehi, o);
        elo += __shfl_xor_sync(0xffffffffu, elo, o);
    }
    if (lane == 0 && (ehi | elo)) { red_add_s64(p.out + pk_ehi(d), ehi); red_add_s64(p.out + pk_ehi(d) + 1, elo); }
    finish_changed(d, p.out, ch);
}

// ------------------------------------------------------------------
// Sorted engine for large shards (n >= AAKM_SORTED_MIN_ROWS): rows are
// bucketed by label, then each warp sums a chunk of <= SEG_ROWS rows of one
// cluster in fp64 registers (lanes over d) and issues d atomics per chunk
// instead of d per row.  X is read exactly once, as contiguous row segments;
// the energy uses the chunk's centroid kept in registers.
//   k_hist     N_j (block histograms in smem) + #changed + label check
//   k_scan_a   per cluster: N_j -> packed, per-(block, cluster) offsets within the cluster
//   k_scan_b   exclusive scans over clusters, chunk counts, chunk -> cluster map
//   k_scatter  perm[offset_j + rank] = row (warp-aggregated cursors)
//   k_segsum   S_j += sum of the chunk's rows, E += sum (x - c_j)^2

constexpr int SEG_ROWS = 256;

__device__ void finish_changed(const Dev& d, long long* out, long long ch) {
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
        out[pk_ch(d)] += bc;                              // changed (packed was zeroed)
        d.st->hist_ctr = 0;
    }
}

// Block b histograms its contiguous row range [b*R, (b+1)*R) into smem and
// stores it to seg_bh[b][K]; k_scan_a/b turn counts into per-(block, cluster)
// base offsets, and k_scatter re-walks the same rows placing each at
// base + local rank (shared-memory counters): no global atomics on the
// contended per-cluster cursors.
__device__ __forceinline__ void block_rows(const Dev& d, long long& r0, long long& r1) {
    const long long per = (d.n + gridDim.x - 1) / gridDim.x;
    r0 = (long long)blockIdx.x * per;
    r1 = min(d.n, r0 + per);
}

__global__ void __launch_bounds__(1024) k_hist(Dev d, GEval g) {
    if (!geval_active(d, g)) return;
    const Pick p = pick(d, g);
    extern __shared__ int hs[];
    const int K = d.K;
    for (int j = threadIdx.x; j < K; j += blockDim.x) hs[j] = 0;
    __syncthreads();
    long long r0, r1;
    block_rows(d, r0, r1);
    long long ch = 0;
    int bad = 0;
    // 4 labels per thread per step (more loads in flight: the pass is latency-bound)
    const long long nv = (r1 - r0) / 4;
    for (long long v = threadIdx.x; v < nv; v += blockDim.x) {
        const long long i = r0 + 4 * v;
        int l4[4], p4[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) { l4[u] = p.lab[i + u]; p4[u] = p.prev ? p.prev[i + u] : l4[u]; }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int j = l4[u];
            if (j < 0 || j >= K) { bad = 1; continue; }
            ch += (p4[u] != j);
            atomicAdd(&hs[j], 1);
        }
    }
    for (long long i = r0 + 4 * nv + threadIdx.x; i < r1; i += blockDim.x) {
        const int j = p.lab[i];
        if (j < 0 || j >= K) { bad = 1; continue; }
        if (p.prev) ch += (p.prev[i] != j);
        atomicAdd(&hs[j], 1);
    }
    if (bad) d.st->label_error = 1;
    __syncthreads();
    int* bh = d.seg_bh + (long long)blockIdx.x * K;
    for (int j = threadIdx.x; j < K; j += blockDim.x) bh[j] = hs[j];
    finish_changed(d, p.out, ch);
}

// Phase A (one thread per cluster, many blocks): N_j = sum over row blocks, and
// the per-(block, cluster) offsets within cluster j (exclusive scan over blocks).
__global__ void __launch_bounds__(256) k_scan_a(Dev d, GEval g, int nblk) {
    if (!geval_active(d, g)) return;
    const Pick p = pick(d, g);
    const int K = d.K;
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= K) return;
    long long o = 0;
    int b = 0;
    for (; b + 8 <= nblk; b += 8) {
        int t[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) t[u] = d.seg_bh[(long long)(b + u) * K + j];
#pragma unroll
        for (int u = 0; u < 8; ++u) { d.seg_bh[(long long)(b + u) * K + j] = (int)o; o += t[u]; }
    }
    for (; b < nblk; ++b) {
        const int t = d.seg_bh[(long long)b * K + j];
        d.seg_bh[(long long)b * K + j] = (int)o;
        o += t;
    }
    d.seg_off[j] = (int)o;                               // count for now; phase B makes it an offset
    p.out[pk_n(d) + j] = o;                              // N_j
}

// Phase B (one block): exclusive scans over clusters of the counts and of the
// chunk counts, chunk -> cluster map.  k_scatter adds seg_off[j] to the bases.
__global__ void __launch_bounds__(1024) k_scan_b(Dev d, GEval g) {
    if (!geval_active(d, g)) return;
    const int K = d.K;
    __shared__ long long wsum[2][32];
    __shared__ long long carry[2];
    if (threadIdx.x == 0) { carry[0] = 0; carry[1] = 0; }
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int base = 0; base < K; base += blockDim.x) {
        const int j = base + threadIdx.x;
        const long long c = j < K ? d.seg_off[j] : 0;
        const long long nc = (c + SEG_ROWS - 1) / SEG_ROWS;
        long long a = c, bb = nc;
        for (int o = 1; o < 32; o <<= 1) {
            const long long ta = __shfl_up_sync(0xffffffffu, a, o), tb = __shfl_up_sync(0xffffffffu, bb, o);
            if (lane >= o) { a += ta; bb += tb; }
        }
        if (lane == 31) { wsum[0][w] = a; wsum[1][w] = bb; }
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
        const long long pb = (w ? wsum[1][w - 1] : 0) + bb - nc + carry[1];
        __syncthreads();                                 // every thread has read its count
        if (j < K) {
            d.seg_off[j] = (int)pa;
            d.seg_chunk[j] = (int)pb;
            for (long long q = 0; q < nc; ++q) d.seg_cmap[pb + q] = j;
        }
        if (threadIdx.x == blockDim.x - 1) { carry[0] = pa + c; carry[1] = pb + nc; }
        __syncthreads();
    }
    if (threadIdx.x == 0) { d.seg_off[K] = (int)carry[0]; d.seg_chunk[K] = (int)carry[1]; }
}

__global__ void __launch_bounds__(1024) k_scatter(Dev d, GEval g) {
    if (!geval_active(d, g)) return;
    const Pick p = pick(d, g);
    extern __shared__ int cur[];
    const int K = d.K;
    const int* bh = d.seg_bh + (long long)blockIdx.x * K;
    for (int j = threadIdx.x; j < K; j += blockDim.x) cur[j] = bh[j] + d.seg_off[j];
    __syncthreads();
    long long r0, r1;
    block_rows(d, r0, r1);
    const long long nv = (r1 - r0) / 4;
    for (long long v = threadIdx.x; v < nv; v += blockDim.x) {
        const long long i = r0 + 4 * v;
        int l4[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) l4[u] = p.lab[i + u];
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (l4[u] >= 0 && l4[u] < K) d.perm[atomicAdd(&cur[l4[u]], 1)] = (int)(i + u);
    }
    for (long long i = r0 + 4 * nv + threadIdx.x; i < r1; i += blockDim.x) {
        const int j = p.lab[i];
        if (j < 0 || j >= K) continue;
        d.perm[atomicAdd(&cur[j], 1)] = (int)i;
    }
}

template <int V>   // floats per lane: d <= 32 * V
__global__ void __launch_bounds__(256) k_segsum(Dev d, GEval g) {
    if (!geval_active(d, g)) return;
    const Pick p = pick(d, g);
    const int D = d.d, K = d.K;
    const long long KD = (long long)K * D;
    const int lane = threadIdx.x & 31;
    const long long nchunks = d.seg_chunk[K];
    const float sc = d.fx_scale;
    const double q = energy_q(d);
    long long ehi = 0, elo = 0;
    for (long long w = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); w < nchunks;
         w += (long long)gridDim.x * (blockDim.x >> 5)) {
        const int j = d.seg_cmap[w];
        const long long r0 = d.seg_off[j] + (w - d.seg_chunk[j]) * SEG_ROWS;
        const int cnt = (int)min((long long)SEG_ROWS, (long long)d.seg_off[j + 1] - r0);
        // the chunk's row ids, 8 per lane, fetched up front (one round trip)
        int rid[SEG_ROWS / 32];
#pragma unroll
        for (int u = 0; u < SEG_ROWS / 32; ++u) {
            const int qi = u * 32 + lane;
            rid[u] = qi < cnt ? d.perm[r0 + qi] : -1;
        }
        int hi[V], lo[V];                         // <= 256 rows per chunk: int32 cannot overflow
        float cj[V];
#pragma unroll
        for (int v = 0; v < V; ++v) {
            hi[v] = 0; lo[v] = 0;
            const int k = lane + 32 * v;
            cj[v] = k < D ? __ldg(p.C + (long long)j * D + k) : 0.f;
        }
#pragma unroll
        for (int u = 0; u < SEG_ROWS / 32; ++u) {
            if (u * 32 < cnt) {                   // predicate, not break: keeps rid[] in registers
            float xv[8][V];
#pragma unroll
            for (int b8 = 0; b8 < 32; b8 += 8) {
#pragma unroll
                for (int t = 0; t < 8; ++t) {
                    const int row = __shfl_sync(0xffffffffu, rid[u], b8 + t);
#pragma unroll
                    for (int v = 0; v < V; ++v) {
                        const int k = lane + 32 * v;
                        xv[t][v] = (row >= 0 && k < D) ? __ldcs(d.X + (long long)row * D + k) : 0.f;
                    }
                }
#pragma unroll
                for (int t = 0; t < 8; ++t) {
                    double e = 0.0;
#pragma unroll
                    for (int v = 0; v < V; ++v) {
                        fx_add(xv[t][v], sc, hi[v], lo[v]);   // zeros add nothing
                        const int k = lane + 32 * v;
                        if (k < D) { const double df = (double)xv[t][v] - (double)cj[v]; e = fma(df, df, e); }
                    }
                    for (int o = 16; o; o >>= 1) e += __shfl_xor_sync(0xffffffffu, e, o);
                    const int row = __shfl_sync(0xffffffffu, rid[u], b8 + t);
                    if (lane == 0 && row >= 0) energy_add(e, q, ehi, elo);
                }
            }
            }
        }
#pragma unroll
        for (int v = 0; v < V; ++v) {
            const int k = lane + 32 * v;
            if (k < D) {
                red_add_s64(p.out + (long long)j * D + k, hi[v]);
                red_add_s64(p.out + KD + (long long)j * D + k, lo[v]);
            }
        }
    }
    if (lane == 0 && (ehi | elo)) { red_add_s64(p.out + pk_ehi(d), ehi); red_add_s64(p.out + pk_ehi(d) + 1, elo); }
}

// float4 variant (d = 4 * LPR, LPR in {1,2,4,8,16,32}): LPR lanes cover one
// row, RPW = 32 / LPR rows per warp instruction, 16 rows in flight per warp.
template <int LPR>
__global__ void __launch_bounds__(256) k_segsum4(Dev d, GEval g) {
    if (!geval_active(d, g)) return;
    constexpr int RPW = 32 / LPR;
    constexpr int U = (16 / RPW) > 0 ? 16 / RPW : 1;     // instructions per round
    constexpr int ROUND = U * RPW;                       // rows per round (16, or 32 when RPW = 32)
    const Pick p = pick(d, g);
    const int D = d.d, K = d.K;
    const long long KD = (long long)K * D;
    const int lane = threadIdx.x & 31;
    const int h = lane / LPR, c4i = lane % LPR;          // row slot within the instruction, float4 index
    const long long nchunks = d.seg_chunk[K];
    const float4* X4 = reinterpret_cast<const float4*>(d.X);
    const float sc = d.fx_scale;
    const double q = energy_q(d);
    long long ehi = 0, elo = 0;
    for (long long w = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); w < nchunks;
         w += (long long)gridDim.x * (blockDim.x >> 5)) {
        const int j = d.seg_cmap[w];
        const long long r0 = d.seg_off[j] + (w - d.seg_chunk[j]) * SEG_ROWS;
        const int cnt = (int)min((long long)SEG_ROWS, (long long)d.seg_off[j + 1] - r0);
        int rid[SEG_ROWS / 32];
#pragma unroll
        for (int t = 0; t < SEG_ROWS / 32; ++t) {
            const int qi = t * 32 + lane;
            rid[t] = qi < cnt ? d.perm[r0 + qi] : -1;
        }
        const float4 c = __ldg(reinterpret_cast<const float4*>(p.C + (long long)j * D) + c4i);
        const double cx = c.x, cy = c.y, cz = c.z, cw = c.w;
        // fixed-point parts of the 4 coordinates, int32 per chunk (<= 256 rows / lane)
        int h0 = 0, h1 = 0, h2 = 0, h3 = 0, l0 = 0, l1 = 0, l2 = 0, l3 = 0;
#pragma unroll
        for (int t = 0; t < SEG_ROWS / 32; ++t) {
            if (t * 32 < cnt) {
#pragma unroll
                for (int r = 0; r < 32; r += ROUND) {
                    float4 xv[U];
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const int rw = __shfl_sync(0xffffffffu, rid[t], (r + u * RPW + h) & 31);
                        xv[u] = rw >= 0 ? __ldcs(X4 + (long long)rw * LPR + c4i) : make_float4(0.f, 0.f, 0.f, 0.f);
                    }
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        fx_add(xv[u].x, sc, h0, l0); fx_add(xv[u].y, sc, h1, l1);
                        fx_add(xv[u].z, sc, h2, l2); fx_add(xv[u].w, sc, h3, l3);
                        // e_i by direct differences: 4 coordinates here, then the row's LPR lanes
                        double df = (double)xv[u].x - cx, e = df * df;
                        df = (double)xv[u].y - cy; e = fma(df, df, e);
                        df = (double)xv[u].z - cz; e = fma(df, df, e);
                        df = (double)xv[u].w - cw; e = fma(df, df, e);
#pragma unroll
                        for (int o = 1; o < LPR; o <<= 1) e += __shfl_xor_sync(0xffffffffu, e, o);
                        const int rw = __shfl_sync(0xffffffffu, rid[t], (r + u * RPW + h) & 31);
                        if (c4i == 0 && rw >= 0) energy_add(e, q, ehi, elo);
                    }
                }
            }
        }
        // combine the RPW row slots (lanes with equal c4i): exact int64 sums
        long long s[8] = {h0, h1, h2, h3, l0, l1, l2, l3};
#pragma unroll
        for (int o = LPR; o < 32; o <<= 1) {
#pragma unroll
            for (int qq = 0; qq < 8; ++qq) s[qq] += __shfl_xor_sync(0xffffffffu, s[qq], o);
        }
        if (h == 0) {
            long long* oh = p.out + (long long)j * D + 4 * c4i;
            long long* ol = oh + KD;
#pragma unroll
            for (int qq = 0; qq < 4; ++qq) { red_add_s64(oh + qq, s[qq]); red_add_s64(ol + qq, s[4 + qq]); }
        }
    }
    for (int o = 16; o; o >>= 1) {
        ehi += __shfl_xor_sync(0xffffffffu, ehi, o);
        elo += __shfl_xor_sync(0xffffffffu, elo, o);
    }
    if (lane == 0 && (ehi | elo)) { red_add_s64(p.out + pk_ehi(d), ehi); red_add_s64(p.out + pk_ehi(d) + 1, elo); }
}

cudaError_t setup_update() {
    cudaError_t e = cudaFuncSetAttribute(k_hist, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * AAKM_SORTED_MAX_K);
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(k_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * AAKM_SORTED_MAX_K);
}

// Chosen from global quantities so every rank runs the same per-row energy order
// (E is then identical for every rank count).
bool update_sorted(long long n_global, int dd, int K) {
    return n_global >= AAKM_SORTED_MIN_ROWS && dd <= 128 && K <= AAKM_SORTED_MAX_K;
}

int launch_update(const Dev& d, const GEval& g, cudaStream_t s) {
    if (!d.upd_sorted) {
        k_update<<<d.upd_blocks, 256, 0, s>>>(d, g);
        return 1;
    }
    const size_t hs = (size_t)d.K * 4;
    k_hist<<<AAKM_SEG_BLOCKS, 1024, hs, s>>>(d, g);
    k_scan_a<<<(d.K + 255) / 256, 256, 0, s>>>(d, g, AAKM_SEG_BLOCKS);
    k_scan_b<<<1, 1024, 0, s>>>(d, g);
    k_scatter<<<AAKM_SEG_BLOCKS, 1024, hs, s>>>(d, g);
    if (d.d % 4 == 0 && (d.d / 4) <= 32 && ((d.d / 4) & (d.d / 4 - 1)) == 0) {
        switch (d.d / 4) {
            case 1: k_segsum4<1><<<d.upd_blocks, 256, 0, s>>>(d, g); return 5;
            case 2: k_segsum4<2><<<d.upd_blocks, 256, 0, s>>>(d, g); return 5;
            case 4: k_segsum4<4><<<d.upd_blocks, 256, 0, s>>>(d, g); return 5;
            case 8: k_segsum4<8><<<d.upd_blocks, 256, 0, s>>>(d, g); return 5;
            case 16: k_segsum4<16><<<d.upd_blocks, 256, 0, s>>>(d, g); return 5;
            default: k_segsum4<32><<<d.upd_blocks, 256, 0, s>>>(d, g); return 5;
        }
    }
    const int V = (d.d + 31) / 32;
    switch (V) {
        case 1: k_segsum<1><<<d.upd_blocks, 256, 0, s>>>(d, g); break;
        case 2: k_segsum<2><<<d.upd_blocks, 256, 0, s>>>(d, g); break;
        case 3: k_segsum<3><<<d.upd_blocks, 256, 0, s>>>(d, g); break;
        default: k_segsum<4><<<d.upd_blocks, 256, 0, s>>>(d, g); break;
    }
    return 5;
}

// kmeans_update API: G = S / N (empty -> C_prev row, R-A15), counts.
__global__ void k_update_G(Dev d, const long long* packed, const float* Cprev, float* G, long long* counts) {
    const long long KD = (long long)d.K * d.d;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < KD; e += (long long)gridDim.x * blockDim.x) {
        const long long j = e / d.d;
        const long long nj = packed[pk_n(d) + j];
        G[e] = nj > 0 ? (float)(fx_value(packed[e], packed[KD + e], d.fx_inv) / (double)nj) : Cprev[e];
        if (counts && e % d.d == 0) counts[j] = nj;
    }
}

void launch_update_G(const Dev& d, const long long* packed, const float* Cprev, float* G,
                     long long* counts, cudaStream_t s) {
    long long KD = (long long)d.K * d.d;
    int blocks = (int)((KD + 255) / 256);
    if (blocks > 1184) blocks = 1184;
    k_update_G<<<blocks, 256, 0, s>>>(d, packed, Cprev, G, counts);
}

}  // namespace aakm

namespace aakm {

// ------------------------------------------------------------------
// E from its reduced fixed-point parts (after the allreduce): identical bytes on
// every rank and for every rank count.
__global__ void k_energy(Dev d, GEval g) {
    if (!geval_active(d, g)) return;
    const Pick p = pick(d, g);
    const double q = energy_q(d);
    const long long* e = p.out + pk_ehi(d);
    p.out[pk_e(d)] = __double_as_longlong(((double)e[0] + (double)e[1] * 9.313225746154785e-10) / q);
}

void launch_energy(const Dev& d, const GEval& g, cudaStream_t s) { k_energy<<<1, 1, 0, s>>>(d, g); }

// kmeans_update_partials: this rank's unreduced [S | N | E_local | changed] as doubles.
__global__ void k_partials_out(Dev d, const long long* pk, double* out) {
    const long long KD = (long long)d.K * d.d;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < KD; e += (long long)gridDim.x * blockDim.x)
        out[e] = fx_value(pk[e], pk[KD + e], d.fx_inv);
    for (long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x; j < d.K; j += (long long)gridDim.x * blockDim.x)
        out[KD + j] = (double)pk[pk_n(d) + j];
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        const long long* e = pk + pk_ehi(d);
        out[KD + d.K] = ((double)e[0] + (double)e[1] * 9.313225746154785e-10) / energy_q(d);
        out[KD + d.K + 1] = (double)pk[pk_ch(d)];
    }
}

void launch_partials_out(const Dev& d, const long long* packed, const float* C, double* out, cudaStream_t s) {
    (void)C;
    k_partials_out<<<64, 256, 0, s>>>(d, packed, out);
}

// ------------------------------------------------------------------ create-time statistics of X
// out4[0] = max |x| (float bits), out4[1] = max ||x_i||^2 (float bits, rounded up)
__global__ void k_xstats_max(const float* X, long long n, int D, unsigned int* out) {
    const int lane = threadIdx.x & 31;
    float am = 0.f, nm = 0.f;
    for (long long i = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n;
         i += ((long long)gridDim.x * blockDim.x) >> 5) {
        double s = 0.0;
        for (int k = lane; k < D; k += 32) {
            const float v = X[i * D + k];
            am = fmaxf(am, fabsf(v));
            s = fma((double)v, (double)v, s);
        }
        for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        nm = fmaxf(nm, __double2float_ru(s));
    }
    for (int o = 16; o; o >>= 1) am = fmaxf(am, __shfl_xor_sync(0xffffffffu, am, o));
    if (lane == 0) { atomicMax(out, __float_as_uint(am)); atomicMax(out + 1, __float_as_uint(nm)); }
}

void launch_xstats_max(const float* X, long long n, int d, unsigned int* out, cudaStream_t s) {
    if (n > 0) k_xstats_max<<<592, 256, 0, s>>>(X, n, d, out);
}

}  // namespace aakm
