// refine.cu -- exact fp64 re-decision of near-tie rows.
//
// The fp32 / 3xTF32 assignment engines flag every row whose two best computed
// scores are within the engine's rigorous error bound.  For those rows the
// argmin of Eq. (3) is recomputed here from the definition,
// D_ij = sum_k (x_ik - c_jk)^2 by direct differences in fp64, k ascending,
// with lowest-index tie-breaking (reading R-A16).  Rounding is forced with
// __d*_rn intrinsics so no FMA contraction changes the result.
//
// Two phases per flagged row (one warp per row):
//  1. fp32 candidate filter: the same FFMA-chain score on fl32(C) as assign_simt.cu for
//     every centroid; with the rigorous fp32 bound e, only centroids with
//     score <= min score + 2e can be the exact argmin;
//  2. fp64 distances to the fp64 centroids for those candidates only.
#include "aakm_dev.cuh"

namespace aakm {

__device__ __forceinline__ double exact_sqdist(const float* __restrict__ x, const double* __restrict__ c, int D) {
    double acc = 0.0;
    for (int k = 0; k < D; ++k) {
        double diff = __dsub_rn((double)x[k], c[k]);
        acc = __dadd_rn(acc, __dmul_rn(diff, diff));
    }
    return acc;
}

// dynamic smem: per warp, x (fp32, d floats) + candidate list (CAND ints)
constexpr int CAND = 64;

__global__ void __launch_bounds__(256) k_refine(Dev d, GEval g, long long first) {
    if (!geval_active(d, g)) return;
    extern __shared__ float4 smem4[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int D = d.d;
    float* xw = reinterpret_cast<float*>(smem4) + (size_t)warp * (D + CAND);
    int* cand = reinterpret_cast<int*>(xw + D);
    int* lab_out = g.lab_out ? g.lab_out : d.lab[d.st->cur];
    const long long nflag = d.flag_count[g.branch];
    const long long gw = first + (long long)blockIdx.x * 8 + warp;
    const long long nw = (long long)gridDim.x * 8;
    for (long long f = gw; f < nflag; f += nw) {
        const long long row = d.flag_rows[f];
        for (int k = lane; k < D; k += 32) xw[k] = d.X[row * D + k];
        __syncwarp();
        float xn = 0.f;
        for (int k = 0; k < D; ++k) xn = fmaf(xw[k], xw[k], xn);
        // phase 1: fp32 scores and their minimum
        float best = INFINITY;
        for (int j = lane; j < d.K; j += 32) {
            const float* c = d.C32 + (long long)j * D;
            float s = d.cn[j];
            for (int k = 0; k < D; ++k) s = fmaf(xw[k], -2.0f * c[k], s);
            best = fminf(best, s);
        }
        for (int o = 16; o; o >>= 1) best = fminf(best, __shfl_xor_sync(0xffffffffu, best, o));
        const float cmax2 = __uint_as_float(d.st->cmax2_bits);
        // 2e with e the per-score bound of the fp32 chain on fl32(C) (the SIMT engine's gamma)
        const float lim = best + 8.0f * (float)(D + 3) * 5.9604645e-8f * (xn + cmax2);
        // phase 2: exact fp64 on candidates (recompute s; collect in smem, overflow -> all)
        int ncand = 0;
        bool overflow = false;
        for (int j0 = 0; j0 < d.K; j0 += 32) {
            int j = j0 + lane;
            bool isc = false;
            if (j < d.K) {
                const float* c = d.C32 + (long long)j * D;
                float s = d.cn[j];
                for (int k = 0; k < D; ++k) s = fmaf(xw[k], -2.0f * c[k], s);
                isc = s <= lim;
            }
            unsigned m = __ballot_sync(0xffffffffu, isc);
            int pos = ncand + __popc(m & ((1u << lane) - 1));
            if (isc && pos < CAND) cand[pos] = j;
            ncand += __popc(m);
        }
        __syncwarp();
        if (ncand > CAND) overflow = true;
        double bd = INFINITY;
        int bj = 0x7fffffff;
        const int nc = overflow ? d.K : ncand;
        for (int q = lane; q < nc; q += 32) {
            int j = overflow ? q : cand[q];
            double v = exact_sqdist(xw, d.C + (long long)j * D, D);
            if (v < bd || (v == bd && j < bj)) { bd = v; bj = j; }
        }
        for (int o = 16; o; o >>= 1) {
            double ov = __shfl_xor_sync(0xffffffffu, bd, o);
            int oj = __shfl_xor_sync(0xffffffffu, bj, o);
            if (ov < bd || (ov == bd && oj < bj)) { bd = ov; bj = oj; }
        }
        if (lane == 0) {
            lab_out[row] = bj;
            if (d.pj2) { d.pj2[row] = -1; d.ub[row] = INFINITY; }   // bounded: re-score next time
        }
        __syncwarp();
    }
}

cudaError_t setup_refine() {
    return cudaFuncSetAttribute(k_refine, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * (4096 + CAND) * 4);
}

int launch_refine(const Dev& d, const GEval& g, cudaStream_t s, long long first) {
    size_t smem = (size_t)8 * (d.d + CAND) * 4;
    k_refine<<<296, 256, smem, s>>>(d, g, first);
    return 1;
}

}  // namespace aakm
