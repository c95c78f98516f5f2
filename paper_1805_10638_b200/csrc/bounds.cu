// bounds.cu -- Hamerly-bounded assignment for the 2xFP16 tensor engine (f2).
//
// The paper's Assignment-Step is Hamerly-pruned: per sample
// an upper bound u_i on the distance to its own centroid and a lower bound l_i
// on the distance to every other one.  When the centroids move by
// s_j = ||c_j - c_ref_j||, u_i + s_{rho_i} and l_i - max_j s_j remain bounds, and
// u_i < l_i proves the label is unchanged (the exact argmin is still rho_i).
// Here the surviving rows are not scanned one by one: the unproven rows form a
// gathered list that the tensor engine runs in MODE 2, which writes fresh
// bounds (from its exact window keys and error bound) for every row it scores.
//   k_shift   s_j and max_j s_j for the set about to be assigned; C_ref <- it
//   k_bounds  per row: the Hamerly test; proven rows keep (copy) their label and
//             move their bounds, the rest are appended to act_rows
// AA jumps: branch A's shifts are measured from the previous pass's assigned
// set; the state is snapshotted first (k_bnd_save), and a fallback B (after a
// rejected jump) restores it (k_bnd_restore), so B's shifts are measured from
// that same set, not from the rejected candidate.  All bound arithmetic rounds
// outward.
#include <math.h>

#include "aakm_dev.cuh"

namespace aakm {

__global__ void __launch_bounds__(256) k_shift(Dev d, GEval g) {
    if (!geval_active(d, g)) return;
    DevState* st = d.st;
    const double* C = d.C;
    const int D = d.d;
    const int lane = threadIdx.x & 31;
    float bmax = 0.f;
    for (long long j = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); j < d.K;
         j += (long long)gridDim.x * (blockDim.x >> 5)) {
        double s = 0.0;
        for (int k = lane; k < D; k += 32) {
            const double c = C[j * D + k];
            const double df = c - d.C_ref[j * D + k];
            s = fma(df, df, s);
            d.C_ref[j * D + k] = c;
        }
        for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        const float sh = (float)(sqrt(s) * (1.0 + 1e-12)) * 1.000001f;   // upward
        if (lane == 0) d.shift[j] = sh;
        bmax = fmaxf(bmax, sh);
    }
    for (int o = 16; o; o >>= 1) bmax = fmaxf(bmax, __shfl_xor_sync(0xffffffffu, bmax, o));
    __shared__ float wm[32];
    __shared__ bool last;
    if (lane == 0) wm[threadIdx.x >> 5] = bmax;
    __syncthreads();
    if (threadIdx.x == 0) {
        float m = 0.f;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) m = fmaxf(m, wm[i]);
        atomicMax(&st->shift_tmp, __float_as_uint(m));          // non-negative floats order as uints
        __threadfence();
        last = atomicAdd(&st->shift_ctr, 1u) == gridDim.x - 1;
        if (last) {
            __threadfence();
            st->shift_max_bits = atomicExch(&st->shift_tmp, 0u);
            st->shift_ctr = 0;
            st->bnd_use = st->bnd_ready;                        // bounds valid for this assignment?
            st->bnd_ready = 1;                                  // ... and (fresh or moved) for the next
        }
    }
}

__global__ void __launch_bounds__(256) k_bounds(Dev d, GEval g) {
    if (!geval_active(d, g)) return;
    const DevState* st = d.st;
    if (!st->bnd_use) return;                                   // first assignment: dense
    const float smax = __uint_as_float(st->shift_max_bits);
    const int cur = st->cur;
    int* lab_out = g.lab_out ? g.lab_out : d.lab[cur];
    // labels the bounds refer to: the previous pass's final labels P^{t-1}, for both
    // branches (B restored the snapshot taken before A)
    const int* lab_ref = d.lab[cur ^ 1];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const long long n = d.n;
    // 1024 rows per block step (4 consecutive rows per thread); the unproven rows of
    // a step are appended with ONE atomic per block step, in row order within it
    __shared__ int wcnt[8];
    __shared__ long long sbase;
    constexpr int RPT = 4;
    const long long step = (long long)blockDim.x * RPT;
    // exclusive block prefix of per-thread counts, one atomic on *ctr per block step
    auto block_append = [&](int c, unsigned long long* ctr) -> long long {
        int incl = c;
        for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        if (lane == 31) wcnt[warp] = incl;
        __syncthreads();
        if (threadIdx.x == 0) {
            int tot = 0;
            for (int w = 0; w < (int)(blockDim.x >> 5); ++w) { const int v = wcnt[w]; wcnt[w] = tot; tot += v; }
            sbase = tot ? (long long)atomicAdd(ctr, (unsigned long long)tot) : 0;
        }
        __syncthreads();
        const long long pos = sbase + wcnt[warp] + incl - c;
        __syncthreads();                                        // wcnt / sbase reusable
        return pos;
    };
    for (long long i0 = (long long)blockIdx.x * step; i0 < n; i0 += (long long)gridDim.x * step) {
        const long long ib = i0 + (long long)threadIdx.x * RPT;
        unsigned um = 0, pm = 0;                                // bit k: row ib + k unproven / proven pair
        int pa[RPT], pb2[RPT];
#pragma unroll
        for (int k = 0; k < RPT; ++k) {
            const long long i = ib + k;
            pa[k] = 0; pb2[k] = -1;
            if (i < n) {
                const int a = lab_ref[i];
                const int p2 = d.pj2[i];
                // two-centroid rows: ub bounds both candidates, so it moves with the
                // larger of their shifts; proven, the argmin is one of the two
                const float sh = p2 >= 0 ? fmaxf(d.shift[a], d.shift[p2]) : d.shift[a];
                const float u = __fadd_ru(d.ub[i], sh);
                const float l = __fsub_rd(d.lb[i], smax);
                if (u < l) {
                    d.ub[i] = u;
                    d.lb[i] = l;
                    lab_out[i] = a;
                    if (p2 >= 0) {
                        // two-centroid row: if the last exact decision's distance gap, less
                        // both candidates' shifts (rounded down), still exceeds the fp64
                        // rounding of the distances (1e-9 of u, with room to spare), the
                        // exact argmin is still a -- no pair refine
                        const float gp = d.pgap ? __fsub_rd(__fsub_rd(d.pgap[i], d.shift[a]), d.shift[p2]) : 0.f;
                        if (gp > 1e-9f * u) {
                            d.pgap[i] = gp;
                        } else {
                            pm |= 1u << k; pa[k] = a; pb2[k] = p2;
                        }
                    }
                } else {
                    um |= 1u << k;
                }
            }
        }
        // proven two-centroid rows go straight to the pair list (k_refine_pair)
        if (__syncthreads_or(pm != 0)) {
            long long f = block_append(__popc(pm), (unsigned long long*)&d.pair_count[g.branch]);
#pragma unroll
            for (int k = 0; k < RPT; ++k) {
                if (!(pm & (1u << k))) continue;
                if (f < d.fcap) {
                    d.pair_rows[f] = (int)(ib + k);
                    d.pair_j[f] = make_int2(pa[k], pb2[k]);
                } else {                                        // list full: score the row instead
                    d.ub[ib + k] = INFINITY;
                    um |= 1u << k;
                }
                ++f;
            }
        }
        long long pos = block_append(__popc(um), (unsigned long long*)&d.act_count[g.branch]);
#pragma unroll
        for (int k = 0; k < RPT; ++k)
            if (um & (1u << k)) d.act_rows[pos++] = (int)(ib + k);
    }
}

// branch A: snapshot the bounds state; branch B (rejection only): restore it
__global__ void __launch_bounds__(256) k_bnd_save(Dev d, GEval g, int restore) {
    if (!geval_active(d, g)) return;
    if (!restore && d.st->lloyd) return;                       // a Lloyd candidate is never rejected (R-A9)
    const long long n = d.n, KD = (long long)d.K * d.d;
    const long long st = (long long)gridDim.x * blockDim.x;
    float* ub = restore ? d.ub : d.ub0;
    float* lb = restore ? d.lb : d.lb0;
    int* p2 = restore ? d.pj2 : d.pj20;
    double* cr = restore ? d.C_ref : d.C_ref0;
    const float* ubs = restore ? d.ub0 : d.ub;
    const float* lbs = restore ? d.lb0 : d.lb;
    const int* p2s = restore ? d.pj20 : d.pj2;
    const double* crs = restore ? d.C_ref0 : d.C_ref;
    float* pg = restore ? d.pgap : d.pgap0;
    const float* pgs = restore ? d.pgap0 : d.pgap;
    // 16-B copies (the arrays are 256-B aligned carve regions), scalar tail
    const long long n4 = n >> 2;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += st) {
        reinterpret_cast<float4*>(ub)[i] = reinterpret_cast<const float4*>(ubs)[i];
        reinterpret_cast<float4*>(lb)[i] = reinterpret_cast<const float4*>(lbs)[i];
        reinterpret_cast<int4*>(p2)[i] = reinterpret_cast<const int4*>(p2s)[i];
        if (pg) reinterpret_cast<float4*>(pg)[i] = reinterpret_cast<const float4*>(pgs)[i];
    }
    for (long long i = 4 * n4 + (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += st) {
        ub[i] = ubs[i]; lb[i] = lbs[i]; p2[i] = p2s[i];
        if (pg) pg[i] = pgs[i];
    }
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < KD; i += st) cr[i] = crs[i];
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        if (restore) d.st->bnd_ready = d.st->bnd_ready0;
        else d.st->bnd_ready0 = d.st->bnd_ready;
    }
}

int launch_bounds_prep(const Dev& d, const GEval& g, cudaStream_t s) {
    long long cb = (d.n / 4 + 255) / 256;                 // grid-stride, 16-B copies: 4 blocks per SM suffice
    if (cb > 4 * d.num_sms) cb = 4 * d.num_sms;
    if (cb < 1) cb = 1;
    k_bnd_save<<<(int)cb, 256, 0, s>>>(d, g, g.branch == 1 ? 1 : 0);
    int kb = (int)((d.K + 7) / 8);
    if (kb > 1184) kb = 1184;
    if (kb < 1) kb = 1;
    k_shift<<<kb, 256, 0, s>>>(d, g);
    long long rb = (d.n + 1023) / 1024;                      // 1024 rows per block step
    if (rb > 4 * d.num_sms) rb = 4 * d.num_sms;
    if (rb < 1) rb = 1;
    k_bounds<<<(int)rb, 256, 0, s>>>(d, g);
    return 3;
}

}  // namespace aakm
