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
//          atomic engine (small n): each row by direct differences in fp64 (fixed
//          order), then the same kind of two-part fixed point (energy_q);
//          label-sorted engine: the same quantity through the identity
//          E = sum_i ||x_i||^2 + sum_j (N_j ||c_j||^2 - 2 c_j . S_j)  (DESIGN R-A30),
//          sum_i ||x_i||^2 once per X (k_xstats_max4, fixed point) and the cluster
//          terms from the exact S_j, N_j after the combine (k_energy_x): no fp64
//          work per coordinate in the pass over X
//   changed = #{i : rho_i != rho_i^{prev}}
// X is read once.
#include "aakm_dev.cuh"

namespace aakm {

struct Pick {
    const int* lab;
    const int* prev;
    const double* C;      // C^t (fp64)
    long long* out;       // packed [S_hi | S_lo | N | E_hi | E_lo | E | changed]: where this rank adds
    long long* red;       // the combined vector (after the allreduce / fused flushes): the same
                          // buffer as out unless the rank keeps a local partial (d.partial)
    int fz;               // f4 fused combine: 0 = local adds (+ ncclAllReduce), 1 = multimem, 2 = LSA peers
    long long wo;         // word offset of this branch's buffer in the symmetric window
};

__device__ __forceinline__ Pick pick(const Dev& d, const GEval& g) {
    Pick p;
    const int cur = d.st->cur;
    p.lab = g.lab_out ? g.lab_out : d.lab[cur];
    p.prev = g.prev_mode == 0 ? d.lab[cur ^ 1] : (g.prev_mode == 2 ? g.lab_prev : nullptr);
    p.C = d.C;
    p.out = g.packed_out ? g.packed_out : d.partial[g.branch];   // this rank's partial (= packed[b] unless local)
    p.red = g.packed_out ? g.packed_out : d.packed[g.branch];
    p.fz = g.packed_out ? 0 : d.fused;
    p.wo = g.branch ? d.pk_off1 : 0;
    return p;
}

// Every contribution to the packed vector.  Plain mode: a red.add into this rank's
// buffer (the ranks then combine with ncclAllReduce).  Fused mode (f4, comm.cu): the
// add goes to EVERY rank's replica of the symmetric window at once -- one
// multimem.red through the NVLS multicast address, or one system-scope red per LSA
// peer -- so after the "flushed" device barrier each replica holds the global sum.
__device__ __forceinline__ void pk_add(const Dev& d, const Pick& p, long long idx, long long v) {
    if (p.fz == 0) {
        atomicAdd(reinterpret_cast<unsigned long long*>(p.out + idx), (unsigned long long)v);
    } else if (p.fz == 1) {
        asm volatile("multimem.red.relaxed.sys.global.add.u64 [%0], %1;" ::"l"(d.mc0 + p.wo + idx), "l"(v) : "memory");
    } else {
        for (int r = 0; r < d.lsa_n; ++r)
            asm volatile("red.relaxed.sys.global.add.u64 [%0], %1;" ::"l"(d.lsa0[r] + p.wo + idx), "l"(v) : "memory");
    }
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

__device__ void finish_changed(const Dev& d, const Pick& p, long long ch);

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
                pk_add(d, p, pk_n(d) + j, 1);
            }
            const float* x = d.X + row * D;
            const double* c = p.C + (long long)j * D;
            for (int k = gl; k < D; k += GS) {
                const float xv = __ldcs(x + k);
                int hi = 0, lo = 0;
                fx_add(xv, sc, hi, lo);
                pk_add(d, p, (long long)j * D + k, hi);
                pk_add(d, p, KD + (long long)j * D + k, lo);
                const double df = (double)xv - __ldg(c + k);
                e = fma(df, df, e);
            }
        }
        long long ea = okj ? energy_fx(e * q) : 0;   // this lane's part of e_row
        energy_flush(ea, ehi, elo);
    }
    if (bad) d.st->label_error = 1;
    for (int o = 16; o; o >>= 1) {
        ehi += __shfl_xor_sync(0xffffffffu, ehi, o);
        elo += __shfl_xor_sync(0xffffffffu, elo, o);
    }
    if (lane == 0 && (ehi | elo)) { pk_add(d, p, pk_ehi(d), ehi); pk_add(d, p, pk_ehi(d) + 1, elo); }
    finish_changed(d, p, ch);
}

// ------------------------------------------------------------------
// Sorted engine (n_global >= AAKM_SORTED_MIN_ROWS): rows are bucketed by
// label, then a warp sums a chunk of <= SEG_ROWS rows of one cluster in int32
// fixed-point registers (exact, see fx_add) and issues one int64 atomic per
// coordinate and part per chunk instead of per row.  X is read exactly once;
// E comes from the sums afterwards (k_energy_x).
//   k_hist         N_j (block histograms in smem) + #changed + label check (+ this
//                  rank's sum ||x_i||^2 into the packed vector, block 0)
//   k_scan_a       per cluster: N_j -> packed, per-(block, cluster) offsets
//   k_scan_b       exclusive scans over clusters (row offsets, chunk counts)
//   k_scatter      chunk table {j, first row, rows} + perm[offset_j + rank] = row, written
//                  from per-block counting-sorted sub-tiles (coalesced runs)
//   k_segsum_bulk  d = 4 LPR: rows gathered by TMA tile::gather4 into per-warp
//                  mbarrier rings; S_j += chunk rows
//   k_segsum       other d: lanes over coordinates, the same sums
//   k_energy_x     (after the combine) E from X2, N, S and C

constexpr int SEG_ROWS = 256;

__device__ void finish_changed(const Dev& d, const Pick& p, long long ch) {
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
        pk_add(d, p, pk_ch(d), bc);                       // changed (packed was zeroed)
        d.st->hist_ctr = 0;
    }
}

// Block b histograms its contiguous row range [b*R, (b+1)*R) into smem and
// stores it to seg_bh[b][K]; k_scan_a/b turn counts into per-(block, cluster)
// base offsets, and k_scatter re-walks the same rows placing each at
// base + local rank (shared-memory counters): no global atomics on the
// contended per-cluster cursors.
__device__ __forceinline__ void block_rows(const Dev& d, long long& r0, long long& r1) {
    const long long per = ((d.n + gridDim.x - 1) / gridDim.x + 7) & ~7LL;    // 32-B aligned row ranges
    r0 = (long long)blockIdx.x * per;
    r1 = min(d.n, r0 + per);
}

__global__ void __launch_bounds__(1024) k_hist(Dev d, GEval g) {
    if (!geval_active(d, g)) return;
    if (d.sref && d.st->use_delta) return;                        // the incremental path runs instead
    const Pick p = pick(d, g);
    extern __shared__ int hs[];
    const int K = d.K;
    for (int j = threadIdx.x; j < K; j += blockDim.x) hs[j] = 0;
    __syncthreads();
    long long r0, r1;
    block_rows(d, r0, r1);
    long long ch = 0;
    int bad = 0;
    // 8 labels per thread per step as two 16-B loads (more bytes in flight: the pass is
    // latency-bound); row ranges start 32-B aligned, a caller's unaligned labels go scalar
    const bool vec = ((reinterpret_cast<uintptr_t>(p.lab) | reinterpret_cast<uintptr_t>(p.prev)) & 15) == 0;
    const long long nv = vec ? (r1 - r0) / 8 : 0;
    for (long long v = threadIdx.x; v < nv; v += blockDim.x) {
        const long long i = r0 + 8 * v;
        const int4 la = *reinterpret_cast<const int4*>(p.lab + i), lb = *reinterpret_cast<const int4*>(p.lab + i + 4);
        int4 pa = la, pb = lb;
        if (p.prev) { pa = *reinterpret_cast<const int4*>(p.prev + i); pb = *reinterpret_cast<const int4*>(p.prev + i + 4); }
        const int l8[8] = {la.x, la.y, la.z, la.w, lb.x, lb.y, lb.z, lb.w};
        const int p8[8] = {pa.x, pa.y, pa.z, pa.w, pb.x, pb.y, pb.z, pb.w};
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int j = l8[u];
            if (j < 0 || j >= K) { bad = 1; continue; }
            ch += (p8[u] != j);
            atomicAdd(&hs[j], 1);
        }
    }
    for (long long i = r0 + 8 * nv + threadIdx.x; i < r1; i += blockDim.x) {
        const int j = p.lab[i];
        if (j < 0 || j >= K) { bad = 1; continue; }
        if (p.prev) ch += (p.prev[i] != j);
        atomicAdd(&hs[j], 1);
    }
    if (bad) d.st->label_error = 1;
    if (blockIdx.x == 0 && threadIdx.x == 0 && d.x2) {               // this rank's sum ||x_i||^2 (k_energy_x)
        pk_add(d, p, pk_x2(d), d.x2[0]);
        pk_add(d, p, pk_x2(d) + 1, d.x2[1]);
    }
    __syncthreads();
    int* bh = d.seg_bh + (long long)blockIdx.x * K;
    for (int j = threadIdx.x; j < K; j += blockDim.x) bh[j] = hs[j];
    finish_changed(d, p, ch);
}

// Phase A (one warp per cluster): N_j = sum over the row blocks, and the
// per-(block, cluster) offsets within cluster j (exclusive scan over blocks:
// lane l owns a contiguous run of blocks, then a warp scan of the run sums).
__global__ void __launch_bounds__(256) k_scan_a(Dev d, GEval g, int nblk) {
    if (!geval_active(d, g)) return;
    if (d.sref && d.st->use_delta) return;                        // the incremental path runs instead
    const Pick p = pick(d, g);
    const int K = d.K;
    const int j = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (j >= K) return;
    const int per = (nblk + 31) / 32;                    // <= 16 for the <= 512 row blocks this build uses
    const int b0 = min(nblk, lane * per), b1 = min(nblk, b0 + per);
    int t[16];
    int sum = 0;
#pragma unroll
    for (int u = 0; u < 16; ++u) {
        t[u] = (u < per && b0 + u < b1) ? d.seg_bh[(long long)(b0 + u) * K + j] : 0;
        sum += t[u];
    }
    int inc = sum;
    for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += v;
    }
    int o = inc - sum;
#pragma unroll
    for (int u = 0; u < 16; ++u)
        if (u < per && b0 + u < b1) { d.seg_bh[(long long)(b0 + u) * K + j] = o; o += t[u]; }
    if (lane == 31) {
        d.seg_off[j] = inc;                               // count for now; phase B makes it an offset
        pk_add(d, p, pk_n(d) + j, inc);                   // N_j (the buffer was zeroed)
    }
}

// Phase B (one block): exclusive scans over clusters of the counts and of the
// chunk counts, chunk -> cluster map.  k_scatter adds seg_off[j] to the bases.
__global__ void __launch_bounds__(1024) k_scan_b(Dev d, GEval g) {
    if (!geval_active(d, g)) return;
    if (d.sref && d.st->use_delta) return;                        // the incremental path runs instead
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
        }
        if (threadIdx.x == blockDim.x - 1) { carry[0] = pa + c; carry[1] = pb + nc; }
        __syncthreads();
    }
    if (threadIdx.x == 0) { d.seg_off[K] = (int)carry[0]; d.seg_chunk[K] = (int)carry[1]; }
}

// Rows bucketed by label: block b re-walks its row range (the same ranges as
// k_hist) in sub-tiles of T rows.  A sub-tile is counting-sorted by label in
// shared memory first, then written out in sorted order, so consecutive threads
// store consecutive perm entries of one cluster's run (whole sectors) instead
// of one scattered 4-byte store per row.  Within a cluster the order of rows
// is arbitrary (smem atomics); every sum downstream is order-free.
// Per sub-tile: [ranks: smem atomics] sync [bin scan] sync [stage] sync
// [output + zero the counters + the next sub-tile's label loads] sync.  A row
// travels as one packed word (label << 14 | rank or local row), T <= 2^14.
constexpr int SCAT_RPT = 16;          // rows per thread per sub-tile (T <= SCAT_RPT * BT)
constexpr int SCAT_LB = 14;           // local row / rank bits
static_assert(SCAT_RPT * 1024 <= (1 << SCAT_LB) && AAKM_SORTED_MAX_K <= (1 << (31 - SCAT_LB)), "packed rows");

// cnt[i] (counts) -> exclusive offsets over i < K; base[i] = gcur[i] - offset
// (perm slot of sorted entry q of cluster i is base[i] + q); gcur[i] += count.
// Thread t owns the contiguous bins [t per, (t + 1) per).  Returns the total.
template <int SCAT_BT>
__device__ __forceinline__ int scat_scan(int* cnt, int* gcur, int* base, int K) {
    __shared__ int ws[SCAT_BT / 32];
    const int per = (K + SCAT_BT - 1) / SCAT_BT;            // <= 32
    const int a = threadIdx.x * per, b = min(K, a + per);
    int sum = 0;
    for (int i = a; i < b; ++i) sum += cnt[i];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int inc = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
    }
    if (lane == 31) ws[w] = inc;
    __syncthreads();
    if (w == 0) {
        int x = lane < SCAT_BT / 32 ? ws[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += t;
        }
        if (lane < SCAT_BT / 32) ws[lane] = x;
    }
    __syncthreads();
    int run = inc - sum + (w ? ws[w - 1] : 0);
    const int tot = ws[SCAT_BT / 32 - 1];
    for (int i = a; i < b; ++i) {
        const int c = cnt[i], gc = gcur[i];
        cnt[i] = run;
        base[i] = gc - run;
        gcur[i] = gc + c;
        run += c;
    }
    return tot;
}

// BT = 1024 (one block per SM) or 512 (two per SM, K <= 6144: phases of the two
// blocks overlap)
template <int SCAT_BT>
__global__ void __launch_bounds__(SCAT_BT, SCAT_BT == 512 ? 2 : 1) k_scatter(Dev d, GEval g, int T) {
    if (!geval_active(d, g)) return;
    if (d.sref && d.st->use_delta) return;                        // the incremental path runs instead
    const Pick p = pick(d, g);
    extern __shared__ __align__(16) int scat_sm[];
    const int K = d.K;
    int* cnt = scat_sm;             // K: sub-tile counts -> exclusive offsets
    int* gcur = cnt + K;            // K: next global perm slot of each cluster for this block
    int* base = gcur + K;           // K: output base of the sub-tile's sorted entries
    int* stage = base + K;          // T: packed {label, local row}, sorted by label
    // chunk table {j, first sorted row, rows}: chunk w belongs to the last cluster
    // whose first chunk is <= w (binary search; empty clusters share starts)
    const long long nch = d.seg_chunk[K];
    for (long long w = (long long)blockIdx.x * SCAT_BT + threadIdx.x; w < nch; w += (long long)gridDim.x * SCAT_BT) {
        int lo = 0, hi = K - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (d.seg_chunk[mid] <= w) lo = mid; else hi = mid - 1;
        }
        const long long r0 = d.seg_off[lo] + (w - d.seg_chunk[lo]) * SEG_ROWS;
        d.seg_cmap[w] = make_int4(lo, (int)r0, (int)min((long long)SEG_ROWS, (long long)d.seg_off[lo + 1] - r0), 0);
    }
    const int* bh = d.seg_bh + (long long)blockIdx.x * K;
    for (int j = threadIdx.x; j < K; j += SCAT_BT) { gcur[j] = bh[j] + d.seg_off[j]; cnt[j] = 0; }
    long long r0, r1;
    block_rows(d, r0, r1);
    int pk[SCAT_RPT];
    auto load = [&](long long t0) {
        const int nt = (int)min((long long)T, r1 - t0);
#pragma unroll
        for (int u = 0; u < SCAT_RPT; ++u) {
            const int q = u * SCAT_BT + threadIdx.x;
            pk[u] = q < nt ? __ldcs(p.lab + t0 + q) : -1;
        }
    };
    if (r0 < r1) load(r0);
    __syncthreads();
    for (long long t0 = r0; t0 < r1; t0 += T) {
#pragma unroll
        for (int u = 0; u < SCAT_RPT; ++u) {
            const int j = pk[u];
            pk[u] = (unsigned)j < (unsigned)K ? (j << SCAT_LB) | atomicAdd(&cnt[j], 1) : -1;
        }
        __syncthreads();
        const int nv = scat_scan<SCAT_BT>(cnt, gcur, base, K);
        __syncthreads();
#pragma unroll
        for (int u = 0; u < SCAT_RPT; ++u) {
            if (pk[u] >= 0) {
                const int j = pk[u] >> SCAT_LB;
                stage[cnt[j] + (pk[u] & ((1 << SCAT_LB) - 1))] = (j << SCAT_LB) | (u * SCAT_BT + (int)threadIdx.x);
            }
        }
        __syncthreads();
        if (t0 + T < r1) load(t0 + T);                       // next sub-tile's labels in flight under the output
        for (int j = threadIdx.x; j < K; j += SCAT_BT) cnt[j] = 0;
        int q = threadIdx.x;
        for (; q + 3 * SCAT_BT < nv; q += 4 * SCAT_BT) {
            int e[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) e[u] = stage[q + u * SCAT_BT];
#pragma unroll
            for (int u = 0; u < 4; ++u)
                d.perm[base[e[u] >> SCAT_LB] + q + u * SCAT_BT] = (int)t0 + (e[u] & ((1 << SCAT_LB) - 1));
        }
        for (; q < nv; q += SCAT_BT) {
            const int e = stage[q];
            d.perm[base[e >> SCAT_LB] + q] = (int)t0 + (e & ((1 << SCAT_LB) - 1));
        }
        __syncthreads();
    }
}

constexpr int SCAT_SMEM = 220 * 1024;   // dynamic shared memory of k_scatter (+ its static scan buffer)
// sub-tile rows: a multiple of the block size, <= SCAT_RPT rows per thread, inside
// the shared memory left after the three K-sized arrays
static int scatter_tile(int K, int bt, int per_sm) {
    int T = (SCAT_SMEM / per_sm - 12 * K) / 4;
    T = T / bt * bt;
    return T > SCAT_RPT * bt ? SCAT_RPT * bt : T;
}
// row blocks of the histogram / scatter partition: one per SM.  AAKM_SEG_PER_SM=2
// (A/B runs) takes two 512-thread scatter blocks per SM where the K-sized arrays
// leave room: measured slower (c5 update 0.905 vs 0.870 ms, c3 0.135 vs 0.119)
int seg_blocks_for(int K, int num_sms) {
    static const int env = getenv("AAKM_SEG_PER_SM") ? atoi(getenv("AAKM_SEG_PER_SM")) : 1;
    const int per = env == 2 && scatter_tile(K, 512, 2) >= 4 * 512 ? 2 : 1;
    const int b = per * num_sms;
    return b < AAKM_SEG_BLOCKS_MAX ? b : AAKM_SEG_BLOCKS_MAX;
}

template <int V>   // floats per lane: d <= 32 * V
__global__ void __launch_bounds__(256) k_segsum(Dev d, GEval g) {
    if (!geval_active(d, g)) return;
    if (d.sref && d.st->use_delta) return;                        // the incremental path runs instead
    const Pick p = pick(d, g);
    const int D = d.d, K = d.K;
    const long long KD = (long long)K * D;
    const int lane = threadIdx.x & 31;
    const long long nchunks = d.seg_chunk[K];
    const float sc = d.fx_scale;
    for (long long w = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); w < nchunks;
         w += (long long)gridDim.x * (blockDim.x >> 5)) {
        const int4 ci = d.seg_cmap[w];
        const int j = ci.x;
        const long long r0 = ci.y;
        const int cnt = ci.z;
        // the chunk's row ids, 8 per lane, fetched up front (one round trip)
        int rid[SEG_ROWS / 32];
#pragma unroll
        for (int u = 0; u < SEG_ROWS / 32; ++u) {
            const int qi = u * 32 + lane;
            rid[u] = qi < cnt ? d.perm[r0 + qi] : -1;
        }
        int hi[V], lo[V];                         // <= 256 rows per chunk: int32 cannot overflow
#pragma unroll
        for (int v = 0; v < V; ++v) { hi[v] = 0; lo[v] = 0; }
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
                for (int t = 0; t < 8; ++t)
#pragma unroll
                    for (int v = 0; v < V; ++v) fx_add(xv[t][v], sc, hi[v], lo[v]);   // zeros add nothing
            }
            }
        }
#pragma unroll
        for (int v = 0; v < V; ++v) {
            const int k = lane + 32 * v;
            if (k < D) {
                pk_add(d, p, (long long)j * D + k, hi[v]);
                pk_add(d, p, KD + (long long)j * D + k, lo[v]);
            }
        }
    }
}

// ------------------------------------------------------------------
// Segmented sums with the rows gathered by bulk asynchronous copies (the sorted
// engine's production kernel for d = 4 LPR, LPR a power of two <= 32).
// Each warp walks its chunks (<= SEG_ROWS rows of one cluster j) as items of
// <= SR rows (32, or 16 for d = 128). Producer side: lanes 0..SR/4-1 each start one TMA tile::gather4
// (4 rows by index from the X map)
// into a slot of the warp's NS-deep shared-memory ring, completing on the
// slot's mbarrier; the item's {j, rows, last} go to the slot's record. Row ids
// are loaded two items ahead and chunk records one chunk ahead, so no global
// load sits on the consumer's path. Consumer side: LPR lanes per row (float4
// each), RPW = 32 / LPR rows per shared-memory instruction. The sums are the
// same exact fixed point as the other engines.
#ifndef AAKM_SEG_WMAX
#define AAKM_SEG_WMAX 16
#endif
constexpr int SEG_SMEM = 215040;   // shared memory budget per block

template <int LPR> struct SegBulk {
    // ring depth (items per warp): 3, but 2 for d = 128 (LPR 32), whose 8-KB items
    // otherwise leave too few warps per SM (c4: 2 slots x 11 warps 353 us, 3 x 7 458 us)
    static constexpr int NS = LPR >= 32 ? 2 : 3;
    static constexpr int RB = 16 * LPR;                               // row bytes
    static constexpr int SR = 16;                                      // rows per item
    static constexpr int GP = 4 * RB > 128 ? 4 * RB : 128;            // gather4 group pitch (TMA dst: 128 B aligned)
    static constexpr int SLOT = (SR / 4 * GP + 127) / 128 * 128;       // the item's rows
    static constexpr int WARP = (NS * SLOT + NS * 16 + NS * 8 + 127) / 128 * 128;
    static constexpr int WPB = SEG_SMEM / WARP > AAKM_SEG_WMAX ? AAKM_SEG_WMAX : SEG_SMEM / WARP;
    static constexpr int SMEM = WPB * WARP;
};

__device__ __forceinline__ void sb_init(uint64_t* bar) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(a) : "memory");
}
__device__ __forceinline__ void sb_expect(uint64_t* bar, unsigned bytes) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void sb_copy(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    const unsigned da = (unsigned)__cvta_generic_to_shared(dst);
    const unsigned ba = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(da), "l"(src), "r"(bytes), "r"(ba) : "memory");
}
// 4 rows (box {d, 1} of the X map) -> 4 consecutive d x 4 B rows at dst
__device__ __forceinline__ void sb_gather4(void* dst, const void* map, int r0, int r1, int r2, int r3, uint64_t* bar) {
    const unsigned da = (unsigned)__cvta_generic_to_shared(dst);
    const unsigned ba = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
                 " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                 ::"r"(da), "l"(map), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(ba) : "memory");
}
__device__ __forceinline__ void sb_wait(uint64_t* bar, unsigned phase) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
    unsigned done = 0;
    while (!done) {
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                     : "=r"(done) : "r"(a), "r"(phase) : "memory");
    }
}

// lane g < SR/4 holds the ids of rows 4g..4g+3 of the item (past the end: repeats of its last row)
struct SegItem { int i0, i1, i2, i3, j, nr, last; };

template <int LPR>
__global__ void __launch_bounds__(32 * SegBulk<LPR>::WPB) k_segsum_bulk(Dev d, GEval g) {
    if (!geval_active(d, g)) return;
    if (d.sref && d.st->use_delta) return;                        // the incremental path runs instead
    using SB = SegBulk<LPR>;
    constexpr int RB = SB::RB, RPW = 32 / LPR;
    constexpr int SR = SB::SR;
    constexpr int IT = (SR + RPW - 1) / RPW;                       // consumer instructions per item
    extern __shared__ __align__(128) unsigned char sm[];
    const Pick p = pick(d, g);
    const int D = d.d, K = d.K;
    const long long KD = (long long)K * D;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int h = lane / LPR, c4i = lane % LPR;
    unsigned char* ring = sm + warp * SB::WARP;
    constexpr int SEG_NS = SB::NS;
    int4* rec = reinterpret_cast<int4*>(ring + SEG_NS * SB::SLOT);
    uint64_t* bar = reinterpret_cast<uint64_t*>(rec + SEG_NS);
    if (lane < SEG_NS) sb_init(bar + lane);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    const long long nchunks = d.seg_chunk[K];
    const long long TW = (long long)gridDim.x * SB::WPB;
    const int4 none = make_int4(0, 0, 0, 0);

    // item generator ("ahead" cursor): chunk aw, its record and the next one's
    long long aw = (long long)blockIdx.x * SB::WPB + warp;
    int4 ai = aw < nchunks ? d.seg_cmap[aw] : none;
    int4 an = aw + TW < nchunks ? d.seg_cmap[aw + TW] : none;
    int ast = 0;
    auto gen = [&](SegItem& o) {
        if (aw >= nchunks) { o.nr = 0; o.i0 = o.i1 = o.i2 = o.i3 = 0; o.j = 0; o.last = 0; return; }
        const int base = ast * SR;
        o.j = ai.x;
        o.nr = min(SR, ai.z - base);
        const int* pr = d.perm + ai.y + base;
        const int g4 = 4 * (lane & (SR / 4 - 1)), lst = o.nr - 1;
        o.i0 = pr[min(g4, lst)]; o.i1 = pr[min(g4 + 1, lst)];
        o.i2 = pr[min(g4 + 2, lst)]; o.i3 = pr[min(g4 + 3, lst)];
        o.last = base + SR >= ai.z;
        if (o.last) {
            aw += TW; ai = an; ast = 0;
            an = aw + TW < nchunks ? d.seg_cmap[aw + TW] : none;
        } else {
            ++ast;
        }
    };
    SegItem qa, qb;
    gen(qa);
    gen(qb);
    int ps = 0;                                                        // producer slot
    int inflight = 0;
    auto produce = [&]() {
        if (qa.nr == 0) return;
        uint64_t* b = bar + ps;
        unsigned char* slot = ring + ps * SB::SLOT;
        const int ng = (qa.nr + 3) >> 2;                               // gather4 instructions
        if (lane == 0) { rec[ps] = make_int4(qa.j, qa.nr, qa.last, 0); sb_expect(b, (unsigned)(4 * ng * RB)); }
        __syncwarp();
        if (lane < ng) sb_gather4(slot + lane * SB::GP, d.xg_map, qa.i0, qa.i1, qa.i2, qa.i3, b);
        ps = ps + 1 == SEG_NS ? 0 : ps + 1;
        ++inflight;
        qa = qb;
        gen(qb);
    };
#pragma unroll
    for (int i = 0; i < SEG_NS; ++i) produce();

    const float sc = d.fx_scale;
    unsigned phase = 0;                                                // bit b: parity of slot b
    int cs = 0;                                                        // consumer slot
    int h0 = 0, h1 = 0, h2 = 0, h3 = 0, l0 = 0, l1 = 0, l2 = 0, l3 = 0;
    while (inflight > 0) {
        sb_wait(bar + cs, (phase >> cs) & 1u);
        phase ^= 1u << cs;
        const int4 r = rec[cs];                                        // {j, rows, last}
        const unsigned char* slot = ring + cs * SB::SLOT;
        if (d.dbg & 8) {                                               // AAKM_TC_DBG=8 probe: data movement only
        } else if (RPW <= SR && r.y == SR) {                           // full item (warp-uniform): no masks
#pragma unroll
            for (int i = 0; i < IT; ++i) {
                const int rr = i * RPW + h;
                const unsigned char* a = SB::GP == 4 * RB ? slot + rr * RB + 16 * c4i
                                                          : slot + (rr >> 2) * SB::GP + (rr & 3) * RB + 16 * c4i;
                const float4 xv = *reinterpret_cast<const float4*>(a);
                fx_add(xv.x, sc, h0, l0); fx_add(xv.y, sc, h1, l1);
                fx_add(xv.z, sc, h2, l2); fx_add(xv.w, sc, h3, l3);
            }
        } else {
#pragma unroll
            for (int i = 0; i < IT; ++i) {                             // branch-free: rows past r.y read as 0
                const int rr = i * RPW + h;
                const int ra = RPW > SR ? min(rr, SR - 1) : rr;            // stay inside the slot
                const unsigned char* a = SB::GP == 4 * RB ? slot + ra * RB + 16 * c4i
                                                          : slot + (ra >> 2) * SB::GP + (ra & 3) * RB + 16 * c4i;
                float4 xv = *reinterpret_cast<const float4*>(a);
                if (rr >= r.y) xv = make_float4(0.f, 0.f, 0.f, 0.f);    // adds nothing to the sums
                fx_add(xv.x, sc, h0, l0); fx_add(xv.y, sc, h1, l1);
                fx_add(xv.z, sc, h2, l2); fx_add(xv.w, sc, h3, l3);
            }
        }
        __syncwarp();
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // reads done before the slot refills
        cs = cs + 1 == SEG_NS ? 0 : cs + 1;
        --inflight;
        produce();
        if (!r.z) continue;
        // chunk done: combine the RPW row slots (lanes with equal c4i), exact int64 sums
        long long s8[8] = {h0, h1, h2, h3, l0, l1, l2, l3};
#pragma unroll
        for (int o = LPR; o < 32; o <<= 1) {
#pragma unroll
            for (int t = 0; t < 8; ++t) s8[t] += __shfl_xor_sync(0xffffffffu, s8[t], o);
        }
        if (h == 0) {
            const long long oh = (long long)r.x * D + 4 * c4i;
#pragma unroll
            for (int t = 0; t < 4; ++t) { pk_add(d, p, oh + t, s8[t]); pk_add(d, p, KD + oh + t, s8[4 + t]); }
        }
        h0 = h1 = h2 = h3 = l0 = l1 = l2 = l3 = 0;
    }
}

template <int LPR> static cudaError_t seg_attr() {
    return cudaFuncSetAttribute(k_segsum_bulk<LPR>, cudaFuncAttributeMaxDynamicSharedMemorySize, SegBulk<LPR>::SMEM);
}
template <int LPR> static void seg_launch(const Dev& d, const GEval& g, cudaStream_t s) {
    using SB = SegBulk<LPR>;
    const int per_sm = SB::SMEM <= 113 * 1024 ? 2 : 1;
    k_segsum_bulk<LPR><<<d.num_sms * per_sm, 32 * SB::WPB, SB::SMEM, s>>>(d, g);
}

template <int CPL> __global__ void k_update_priv(Dev d, GEval g);

cudaError_t setup_update() {
    cudaError_t e = cudaFuncSetAttribute(k_hist, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * AAKM_SORTED_MAX_K);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(k_scatter<1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, SCAT_SMEM);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(k_scatter<512>, cudaFuncAttributeMaxDynamicSharedMemorySize, SCAT_SMEM / 2);
    if (e != cudaSuccess) return e;
    for (const void* f : {(const void*)k_update_priv<1>, (const void*)k_update_priv<2>}) {
        e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (2 * AAKM_PRIV_MAX_KD + 4096) * 4);
        if (e != cudaSuccess) return e;
    }
    for (cudaError_t f : {seg_attr<1>(), seg_attr<2>(), seg_attr<4>(), seg_attr<8>(), seg_attr<16>(), seg_attr<32>()})
        if (f != cudaSuccess) return f;
    return cudaSuccess;
}

// Chosen from global quantities so every rank runs the same per-row energy order
// (E is then identical for every rank count).
bool update_sorted(long long n_global, int dd, int K) {
    return n_global >= AAKM_SORTED_MIN_ROWS && dd <= 128 && K <= AAKM_SORTED_MAX_K;
}

// ------------------------------------------------------------------
// Incremental update (one rank, label-sorted engine, d.sref): S(P^t) =
// S(P^{t-1}) + sum over the rows whose label moved of (x_i into the new cluster,
// out of the old one), N likewise.  The fixed-point sums are exact integers, so
// this is bitwise the full recomputation; E comes from the sums (k_energy_x), so
// X is read only for the moved rows.  Late passes move few rows: a pass whose
// moved rows exceed delta_max takes the full sort + segmented sums instead
// (decided on the device per evaluation; the full-path kernels exit early
// otherwise).  S_ref = S(P^{t-1}) is written by k_finalize from the final
// evaluation of every pass and invalidated whenever P^{t-1} or X is replaced.
//   k_delta_scan   moved rows -> list (perm), count; label check; the decision
//   k_delta_copy   packed [S | N] <- S_ref, changed, X2
//   k_delta_add    one warp per moved row: +x into S_new, -x out of S_old (int64)
__global__ void __launch_bounds__(1024) k_delta_scan(Dev d, GEval g) {
    if (!geval_active(d, g)) return;
    DevState* st = d.st;
    if (!st->sref_valid) {
        if (blockIdx.x == 0 && threadIdx.x == 0) { st->use_delta = 0; st->n_upd += 1; }
        return;
    }
    const Pick p = pick(d, g);
    const int K = d.K;
    long long* cnt = d.delta_count + g.branch;
    int bad = 0;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (int)(blockDim.x >> 5);
    // Each block owns a contiguous, 4-aligned row range, read as int4 (4 rows per
    // thread per step: enough loads in flight to stream the two label arrays).
    // Pass 1 counts the moved rows (and checks the labels) without atomics; one
    // counter atomic per block reserves its list slots; pass 2 (only if the whole
    // list can still fit under delta_max) re-reads the labels (L2) and writes the
    // moved rows in row order.
    const long long per = ((d.n + gridDim.x - 1) / gridDim.x + 3) & ~3LL;
    const long long r0 = min(d.n, (long long)blockIdx.x * per), r1 = min(d.n, r0 + per);
    // moved-row mask of rows i0 .. i0 + 3 (bit k: row i0 + k), label check into bad
    auto moved4 = [&](long long i0, int& badv) -> unsigned {
        int j[4], jp[4];
        if (i0 + 3 < r1) {
            const int4 a = *reinterpret_cast<const int4*>(p.lab + i0);
            const int4 b = *reinterpret_cast<const int4*>(p.prev + i0);
            j[0] = a.x; j[1] = a.y; j[2] = a.z; j[3] = a.w;
            jp[0] = b.x; jp[1] = b.y; jp[2] = b.z; jp[3] = b.w;
        } else {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const bool in = i0 + k < r1;
                j[k] = in ? p.lab[i0 + k] : 0;
                jp[k] = in ? p.prev[i0 + k] : 0;
            }
        }
        unsigned mk = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            if (i0 + k >= r1) continue;
            if (j[k] < 0 || j[k] >= K) badv = 1;
            else if (j[k] != jp[k]) mk |= 1u << k;
        }
        return mk;
    };
    int mine = 0;
    for (long long i0 = r0 + 4LL * threadIdx.x; i0 < r1; i0 += 4LL * blockDim.x) mine += __popc(moved4(i0, bad));
    __shared__ int wsum[32];
    __shared__ int itot;
    __shared__ long long bbase;
    __shared__ bool listed;
    for (int o = 16; o; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
    if (lane == 0) wsum[warp] = mine;
    __syncthreads();
    if (threadIdx.x == 0) {
        long long tot = 0;
        for (int w = 0; w < nw; ++w) tot += wsum[w];
        bbase = tot ? (long long)atomicAdd(reinterpret_cast<unsigned long long*>(cnt), (unsigned long long)tot) : 0;
        listed = tot > 0 && bbase + tot <= d.delta_max;           // else the list is not used
    }
    __syncthreads();
    if (listed) {
        long long run = bbase;                                     // next free slot of this block
        int bad2 = 0;
        for (long long b0 = r0; b0 < r1; b0 += 4LL * blockDim.x) {
            const long long i0 = b0 + 4LL * threadIdx.x;
            const unsigned mk = i0 < r1 ? moved4(i0, bad2) : 0u;
            if (!__syncthreads_or(mk != 0)) continue;
            const int c = __popc(mk);
            int x = c;                                             // inclusive scan over the warp
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += y;
            }
            if (lane == 31) wsum[warp] = x;
            __syncthreads();
            if (warp == 0) {                                       // exclusive scan of the warp totals
                const int cw = lane < nw ? wsum[lane] : 0;
                int z = cw;
                for (int o = 1; o < 32; o <<= 1) {
                    const int y = __shfl_up_sync(0xffffffffu, z, o);
                    if (lane >= o) z += y;
                }
                if (lane < nw) wsum[lane] = z - cw;
                if (lane == 31) itot = z;
            }
            __syncthreads();
            long long slot = run + wsum[warp] + (x - c);
            for (unsigned m = mk; m; m &= m - 1) d.perm[slot++] = (int)(i0 + __ffs(m) - 1);
            run += itot;
        }
    }
    if (bad) st->label_error = 1;
    __threadfence();
    __syncthreads();
    __shared__ bool last;
    if (threadIdx.x == 0) last = atomicAdd(&st->delta_ctr, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last || threadIdx.x != 0) return;
    __threadfence();
    st->delta_ctr = 0;
    const long long nm = *(volatile long long*)cnt;
    st->use_delta = nm <= d.delta_max ? 1 : 0;
    st->n_upd += 1;
    if (st->use_delta) { st->n_delta += 1; st->rows_moved += nm; }
}

__global__ void __launch_bounds__(256) k_delta_copy(Dev d, GEval g) {
    if (!geval_active(d, g) || !d.st->use_delta) return;
    const Pick p = pick(d, g);
    const long long W = 2LL * d.K * d.d + d.K;                     // [S_hi | S_lo | N], N at pk_n = 2 K d
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < W; e += (long long)gridDim.x * blockDim.x)
        p.out[e] = d.sref[e];
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        p.out[pk_ch(d)] = d.delta_count[g.branch];                 // changed = the moved rows
        p.out[pk_x2(d)] = d.x2[0];
        p.out[pk_x2(d) + 1] = d.x2[1];
    }
}

__global__ void __launch_bounds__(256) k_delta_add(Dev d, GEval g) {
    if (!geval_active(d, g) || !d.st->use_delta) return;
    const Pick p = pick(d, g);
    const int D = d.d;
    const long long KD = (long long)d.K * D;
    const long long nm = d.delta_count[g.branch];
    const int lane = threadIdx.x & 31;
    const float sc = d.fx_scale;
    for (long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < nm;
         w += ((long long)gridDim.x * blockDim.x) >> 5) {
        const long long row = d.perm[w];
        const long long jn = p.lab[row], jo = p.prev[row];
        for (int k = lane; k < D; k += 32) {
            int hi = 0, lo = 0;
            fx_add(__ldg(d.X + row * D + k), sc, hi, lo);
            red_add_s64(p.out + jn * D + k, hi);
            red_add_s64(p.out + KD + jn * D + k, lo);
            red_add_s64(p.out + jo * D + k, -(long long)hi);
            red_add_s64(p.out + KD + jo * D + k, -(long long)lo);
        }
        if (lane == 0) {
            red_add_s64(p.out + pk_n(d) + jn, 1);
            red_add_s64(p.out + pk_n(d) + jo, -1);
        }
    }
}

// Small K*d shards of the sorted engine (c2: 100 000 x 16, K = 64): one kernel
// instead of sort + segmented sums (5 launches) or the incremental path (3).
// Each block owns <= PRIV_ROWS contiguous rows and accumulates the SAME two-part
// fixed-point integers (fx_add: |hi| <= 2^22, |lo| <= 2^21 per row) into
// shared-memory int32 sums (native shared atomics; 511 rows cannot overflow),
// order-free, so bitwise the sorted engine's S; N_j likewise; then flushes its
// nonzero entries with one int64 red each.  E still comes from the sums
// (k_energy_x).  Lanes are grouped per row (GS = next pow2 >= d): one coalesced
// read per row.
constexpr int PRIV_ROWS = 511;
template <int CPL>                                                  // coordinates per lane: ceil(d / GS)
__global__ void __launch_bounds__(512) k_update_priv(Dev d, GEval g) {
    if (!geval_active(d, g)) return;
    const Pick p = pick(d, g);
    const int D = d.d, K = d.K;
    const int KD = K * D;
    extern __shared__ int sp[];
    int* sh = sp;                                                   // S_hi [K*d]
    int* sl = sp + KD;                                              // S_lo [K*d]
    int* sn = sp + 2 * KD;                                          // N    [K]
    for (int e = threadIdx.x; e < 2 * KD + K; e += blockDim.x) sp[e] = 0;
    __syncthreads();
    int GS = 1;
    while (GS < D && GS < 32) GS <<= 1;
    const int gl = threadIdx.x % GS, gpb = blockDim.x / GS;       // row groups per block
    const long long r0 = min(d.n, (long long)blockIdx.x * PRIV_ROWS), r1 = min(d.n, r0 + PRIV_ROWS);
    const float sc = d.fx_scale;
    long long ch = 0;
    int bad = 0;
    // RB rows per row group and step, every load issued before the first atomic (the
    // loop is latency-bound: one row per step left one global round trip per row)
    constexpr int RB = 8;
    for (long long rb = r0 + threadIdx.x / GS; rb < r1; rb += (long long)RB * gpb) {
        int jr[RB], jp[RB];
        float xv[RB][CPL];
#pragma unroll
        for (int u = 0; u < RB; ++u) {
            const long long row = rb + (long long)u * gpb;
            const bool in = row < r1;
            jr[u] = in ? p.lab[row] : -1;
            jp[u] = in && p.prev ? p.prev[row] : -1;
#pragma unroll
            for (int q = 0; q < CPL; ++q) {
                const int k = gl + q * GS;
                xv[u][q] = in && k < D ? __ldcs(d.X + row * D + k) : 0.f;
            }
        }
#pragma unroll
        for (int u = 0; u < RB; ++u) {
            const long long row = rb + (long long)u * gpb;
            if (row >= r1) break;
            const int j = jr[u];
            if (j < 0 || j >= K) { bad = 1; continue; }          // uniform within the row group
            if (gl == 0) {
                if (p.prev) ch += (jp[u] != j);
                atomicAdd(&sn[j], 1);
            }
#pragma unroll
            for (int q = 0; q < CPL; ++q) {
                const int k = gl + q * GS;
                if (k < D) {
                    int hi = 0, lo = 0;
                    fx_add(xv[u][q], sc, hi, lo);
                    atomicAdd(&sh[j * D + k], hi);
                    atomicAdd(&sl[j * D + k], lo);
                }
            }
        }
    }
    if (bad) d.st->label_error = 1;
    if (blockIdx.x == 0 && threadIdx.x == 0 && d.x2) {            // this rank's sum ||x_i||^2 (k_energy_x)
        pk_add(d, p, pk_x2(d), d.x2[0]);
        pk_add(d, p, pk_x2(d) + 1, d.x2[1]);
    }
    __syncthreads();
    for (int e = threadIdx.x; e < KD; e += blockDim.x) {
        if (sh[e]) pk_add(d, p, e, sh[e]);
        if (sl[e]) pk_add(d, p, (long long)KD + e, sl[e]);
    }
    for (int j = threadIdx.x; j < K; j += blockDim.x)
        if (sn[j]) pk_add(d, p, pk_n(d) + j, sn[j]);
    finish_changed(d, p, ch);
}

int launch_update(const Dev& d, const GEval& g, cudaStream_t s) {
    if (!d.upd_sorted) {
        k_update<<<d.upd_blocks, 256, 0, s>>>(d, g);
        return 1;
    }
    if (d.upd_priv) {
        const size_t sm = (size_t)(2 * d.K * d.d + d.K) * 4;
        const unsigned nb = (unsigned)((d.n + PRIV_ROWS - 1) / PRIV_ROWS);
        if (d.d <= 32) k_update_priv<1><<<nb, 512, sm, s>>>(d, g);
        else k_update_priv<2><<<nb, 512, sm, s>>>(d, g);
        return 1;
    }
    int nl = 0;
    if (d.sref) {                                              // incremental path, decided on the device
        k_delta_scan<<<d.num_sms, 1024, 0, s>>>(d, g);
        k_delta_copy<<<2 * d.num_sms, 256, 0, s>>>(d, g);
        k_delta_add<<<4 * d.num_sms, 256, 0, s>>>(d, g);
        nl = 3;
    }
    const size_t hs = (size_t)d.K * 4;
    const int bt = 1024;
    k_hist<<<d.seg_blocks, bt, hs, s>>>(d, g);
    static_assert(AAKM_SEG_BLOCKS_MAX <= 512, "k_scan_a: <= 16 row blocks per lane");
    k_scan_a<<<(d.K + 7) / 8, 256, 0, s>>>(d, g, d.seg_blocks);
    k_scan_b<<<1, 1024, 0, s>>>(d, g);
    {
        if (d.seg_blocks > d.num_sms) {
            const int T = scatter_tile(d.K, 512, 2);
            k_scatter<512><<<d.seg_blocks, 512, (size_t)(3 * d.K + T) * 4, s>>>(d, g, T);
        } else {
            const int T = scatter_tile(d.K, 1024, 1);
            k_scatter<1024><<<d.seg_blocks, 1024, (size_t)(3 * d.K + T) * 4, s>>>(d, g, T);
        }
    }
    if (d.xg_map) {
        switch (d.d / 4) {
            case 1: seg_launch<1>(d, g, s); return 5 + nl;
            case 2: seg_launch<2>(d, g, s); return 5 + nl;
            case 4: seg_launch<4>(d, g, s); return 5 + nl;
            case 8: seg_launch<8>(d, g, s); return 5 + nl;
            case 16: seg_launch<16>(d, g, s); return 5 + nl;
            default: seg_launch<32>(d, g, s); return 5 + nl;
        }
    }
    const int V = (d.d + 31) / 32;
    switch (V) {
        case 1: k_segsum<1><<<d.upd_blocks, 256, 0, s>>>(d, g); break;
        case 2: k_segsum<2><<<d.upd_blocks, 256, 0, s>>>(d, g); break;
        case 3: k_segsum<3><<<d.upd_blocks, 256, 0, s>>>(d, g); break;
        default: k_segsum<4><<<d.upd_blocks, 256, 0, s>>>(d, g); break;
    }
    return 5 + nl;
}

// kmeans_update API: G = S / N (empty -> C_prev row, R-A15), counts.
__global__ void k_update_G(Dev d, const long long* packed, const double* Cprev, double* G, long long* counts) {
    const long long KD = (long long)d.K * d.d;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < KD; e += (long long)gridDim.x * blockDim.x) {
        const long long j = e / d.d;
        const long long nj = packed[pk_n(d) + j];
        G[e] = nj > 0 ? fx_value(packed[e], packed[KD + e], d.fx_inv) / (double)nj : Cprev[e];
        if (counts && e % d.d == 0) counts[j] = nj;
    }
}

void launch_update_G(const Dev& d, const long long* packed, const double* Cprev, double* G,
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
    const long long* e = p.red + pk_ehi(d);
    p.red[pk_e(d)] = __double_as_longlong(((double)e[0] + (double)e[1] * 9.313225746154785e-10) / q);
}

void launch_energy(const Dev& d, const GEval& g, cudaStream_t s) { k_energy<<<1, 1, 0, s>>>(d, g); }

// The label-sorted engine's energy (DESIGN R-A30): Eq. 1 through the identity
//   E = sum_i ||x_i||^2 + sum_j sum_k (N_j c_jk^2 - 2 c_jk S_jk),
// evaluated from this packed vector (the reduced one, or one rank's partials):
// X2 (k_xstats_max4: each ||x_i||^2 in fp64, rounded to units of 2^x2_e), N_j, the
// exact fixed-point S_jk and the fp64 C.  Each (j, k) term is split into exact fp64
// pieces (two-product), each piece scaled by q (a power of 2) and rounded to the
// E_hi / E_lo grid on its own (efx_add): a fixed function of (N_j, c_jk, S_jk), so
// the integer sums -- and E -- do not depend on order, blocks or rank count.  The
// pieces are computed to ~2^-106 of the term; every piece rounds by <= 2^-31/q.
__device__ __forceinline__ void efx_add(double v, long long& hi, long long& lo) {   // v in units of 1/q
    const double f = floor(v);
    hi += (long long)f;
    lo += __double2ll_rn((v - f) * 1073741824.0);                   // [0, 2^30], exact difference
}
__global__ void __launch_bounds__(256) k_energy_x(Dev d, GEval g) {
    pdl_wait();                                     // PDL: the predecessor's writes are visible
    pdl_trigger();
    if (!geval_active(d, g)) return;
    const Pick p = pick(d, g);
    long long* pk = p.red;                                          // the combined vector (local replica)
    const int D = d.d;
    const long long KD = (long long)d.K * D;
    const double q = energy_q(d);
    const double s22 = d.fx_inv, s44 = d.fx_inv * 2.384185791015625e-07;   // S = Sh 2^(e-22) + Sl 2^(e-44)
    long long hi = 0, lo = 0;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < KD; e += (long long)gridDim.x * blockDim.x) {
        const long long nj = pk[pk_n(d) + e / D];
        if (nj == 0) continue;
        const double c = p.C[e] * q, cq = p.C[e];                   // c q exact (q a power of 2)
        const double N = (double)nj;
        // N c^2 q = N (c2 + c2e) q
        const double c2 = cq * c, c2e = fma(cq, c, -c2);
        const double a1 = N * c2, a1e = fma(N, c2, -a1);
        const double a2 = N * c2e;
        // -2 c S q = -2 c q (Sh s22 + Sl s44)
        const double sh = (double)pk[e] * s22, sl = (double)pk[KD + e] * s44;     // exact
        const double b1 = -2.0 * c * sh, b1e = fma(-2.0 * c, sh, -b1);
        const double b2 = -2.0 * c * sl, b2e = fma(-2.0 * c, sl, -b2);
        efx_add(a1, hi, lo); efx_add(a1e, hi, lo); efx_add(a2, hi, lo);
        efx_add(b1, hi, lo); efx_add(b1e, hi, lo); efx_add(b2, hi, lo); efx_add(b2e, hi, lo);
    }
    for (int o = 16; o; o >>= 1) {
        hi += __shfl_xor_sync(0xffffffffu, hi, o);
        lo += __shfl_xor_sync(0xffffffffu, lo, o);
    }
    if ((threadIdx.x & 31) == 0 && (hi | lo)) {
        atomicAdd(reinterpret_cast<unsigned long long*>(pk + pk_ehi(d)), (unsigned long long)hi);
        atomicAdd(reinterpret_cast<unsigned long long*>(pk + pk_ehi(d) + 1), (unsigned long long)lo);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        // X2 (units 2^x2_e) -> units 2^-30/q = 2^(eb-51): a right shift by eb - 51 - x2_e >= 0, rounded
        int eb = 0;
        frexp(1.0 / q, &eb);                                        // q = 2^(21 - eb): 1/q = 2^(eb-21), frexp -> eb - 20
        const int sh = (eb + 20) - 51 - d.x2_e;
        __int128 v = ((__int128)pk[pk_x2(d)] << 30) + (__int128)pk[pk_x2(d) + 1];
        if (sh > 0) v = (v + ((__int128)1 << (sh - 1))) >> sh;
        atomicAdd(reinterpret_cast<unsigned long long*>(pk + pk_ehi(d)), (unsigned long long)(long long)(v >> 30));
        atomicAdd(reinterpret_cast<unsigned long long*>(pk + pk_ehi(d) + 1), (unsigned long long)(long long)(v & 0x3fffffff));
    }
}

int launch_energy_x(const Dev& d, const GEval& g, cudaStream_t s) {
    if (!d.upd_sorted) return 0;
    long long blocks = ((long long)d.K * d.d + 255) / 256;
    if (blocks > 2 * d.num_sms) blocks = 2 * d.num_sms;
    launch_pdl(k_energy_x, (int)(blocks > 0 ? blocks : 1), 256, 0, s, d, g);
    return 1;
}

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

void launch_partials_out(const Dev& d, const long long* packed, double* out, cudaStream_t s) {
    k_partials_out<<<64, 256, 0, s>>>(d, packed, out);
}

// ------------------------------------------------------------------ create-time statistics of X
// sum_i ||x_i||^2 of the shard for the sorted engine's energy (k_energy_x): every
// x_ik^2 rounded to units of 2^x2_e on its own (to nearest even, by adding
// 1.5 2^52 in one fma: x^2 2^-x2_e < 2^50), so the integer sum is order-free and
// independent of how X is split into rows, ranks or kernels (x2_e = eb0 - 51,
// 2^eb0 > 2 max||x||^2).  Two parts as energy_flush (out[0] units 2^(x2_e+30),
// out[1] units 2^x2_e), out zeroed by the caller.  At create k_x2 computes it;
// a refresh of X gets it from the same pass as the range check (k_xstats_max4).
__device__ __forceinline__ long long x2_units(float x, double s2) {     // s2 = 2^-x2_e
    const double xd = (double)x;
    return __double_as_longlong(fma(xd, xd * s2, 6755399441055744.0)) - 0x4338000000000000LL;
}
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

// The same statistics for d = 4 LPR (LPR a power of two <= 32): LPR lanes per row
// with one 16-B load each, four row groups in flight per warp (the generic kernel
// above reads one float per lane and ran at ~1 TB/s on c5).
template <int LPR>
__global__ void __launch_bounds__(256) k_xstats_max4(const float4* X, long long n, unsigned int* out, long long* x2,
                                                     double s2) {
    constexpr int RPW = 32 / LPR, U = 4;
    const int lane = threadIdx.x & 31, h = lane / LPR, c = lane % LPR;
    float am = 0.f, nm = 0.f;
    long long xh = 0, xl = 0;                                       // sum ||x||^2 (x2_units), two parts
    const long long w0 = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long r0 = w0 * RPW * U; r0 < n; r0 += nw * RPW * U) {
        float4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long long i = r0 + u * RPW + h;
            v[u] = i < n ? __ldcs(X + i * LPR + c) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            am = fmaxf(am, fmaxf(fmaxf(fabsf(v[u].x), fabsf(v[u].y)), fmaxf(fabsf(v[u].z), fabsf(v[u].w))));
            if (x2) {                                               // (rows past n read as zeros)
                const long long a = x2_units(v[u].x, s2) + x2_units(v[u].y, s2) + x2_units(v[u].z, s2) + x2_units(v[u].w, s2);
                xh += a >> 30;
                xl += a & 0x3fffffffLL;
            }
            double s = (double)v[u].x * v[u].x;
            s = fma((double)v[u].y, (double)v[u].y, s);
            s = fma((double)v[u].z, (double)v[u].z, s);
            s = fma((double)v[u].w, (double)v[u].w, s);
#pragma unroll
            for (int o = 1; o < LPR; o <<= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            nm = fmaxf(nm, __double2float_ru(s));
        }
    }
    for (int o = 16; o; o >>= 1) {
        am = fmaxf(am, __shfl_xor_sync(0xffffffffu, am, o));
        nm = fmaxf(nm, __shfl_xor_sync(0xffffffffu, nm, o));
        xh += __shfl_xor_sync(0xffffffffu, xh, o);
        xl += __shfl_xor_sync(0xffffffffu, xl, o);
    }
    if (lane == 0) { atomicMax(out, __float_as_uint(am)); atomicMax(out + 1, __float_as_uint(nm)); }
    if (lane == 0 && x2 && (xh | xl)) {
        atomicAdd(reinterpret_cast<unsigned long long*>(x2), (unsigned long long)xh);
        atomicAdd(reinterpret_cast<unsigned long long*>(x2 + 1), (unsigned long long)xl);
    }
}

int launch_xstats_max(const float* X, long long n, int d, unsigned int* out, cudaStream_t s, long long* x2, int x2_e) {
    if (n <= 0) return 0;
    const bool vec = d % 4 == 0 && d / 4 <= 32 && ((d / 4) & (d / 4 - 1)) == 0 && ((uintptr_t)X & 15) == 0;
    const float4* X4 = reinterpret_cast<const float4*>(X);
    const double s2 = ldexp(1.0, -x2_e);
    if (vec) {
        switch (d / 4) {
            case 1: k_xstats_max4<1><<<1184, 256, 0, s>>>(X4, n, out, x2, s2); return 1;
            case 2: k_xstats_max4<2><<<1184, 256, 0, s>>>(X4, n, out, x2, s2); return 1;
            case 4: k_xstats_max4<4><<<1184, 256, 0, s>>>(X4, n, out, x2, s2); return 1;
            case 8: k_xstats_max4<8><<<1184, 256, 0, s>>>(X4, n, out, x2, s2); return 1;
            case 16: k_xstats_max4<16><<<1184, 256, 0, s>>>(X4, n, out, x2, s2); return 1;
            default: k_xstats_max4<32><<<1184, 256, 0, s>>>(X4, n, out, x2, s2); return 1;
        }
    }
    k_xstats_max<<<592, 256, 0, s>>>(X, n, d, out);
    if (x2) { launch_x2(X, n * d, x2_e, x2, s); return 2; }
    return 1;
}

__global__ void __launch_bounds__(256) k_x2(const float* X, long long count, int x2_e, long long* out) {
    long long hi = 0, lo = 0;
    const double s2 = ldexp(1.0, -x2_e);
    const long long stride = (long long)gridDim.x * blockDim.x;
    const long long n4 = ((reinterpret_cast<uintptr_t>(X) & 15) == 0) ? count / 4 : 0;
    const float4* X4 = reinterpret_cast<const float4*>(X);
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
        const float4 v = __ldcs(X4 + i);
        const long long a = x2_units(v.x, s2) + x2_units(v.y, s2) + x2_units(v.z, s2) + x2_units(v.w, s2);
        hi += a >> 30;
        lo += a & 0x3fffffffLL;
    }
    for (long long i = 4 * n4 + (long long)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) {
        const long long a = x2_units(X[i], s2);
        hi += a >> 30;
        lo += a & 0x3fffffffLL;
    }
    for (int o = 16; o; o >>= 1) {
        hi += __shfl_xor_sync(0xffffffffu, hi, o);
        lo += __shfl_xor_sync(0xffffffffu, lo, o);
    }
    if ((threadIdx.x & 31) == 0 && (hi | lo)) {
        atomicAdd(reinterpret_cast<unsigned long long*>(out), (unsigned long long)hi);
        atomicAdd(reinterpret_cast<unsigned long long*>(out + 1), (unsigned long long)lo);
    }
}

void launch_x2(const float* X, long long count, int x2_e, long long* out, cudaStream_t s) {
    if (count > 0) k_x2<<<1184, 256, 0, s>>>(X, count, x2_e, out);
}

__global__ void k_xcheck(Dev d, const unsigned int* out, unsigned int amax, unsigned int nmax2) {
    if (out[0] > amax || out[1] > nmax2) atomicOr(&d.st->label_error, 2);   // non-negative float bits order as uints
}

void launch_xcheck(const Dev& d, const unsigned int* out, unsigned int amax, unsigned int nmax2, cudaStream_t s) {
    k_xcheck<<<1, 1, 0, s>>>(d, out, amax, nmax2);
}

}  // namespace aakm
