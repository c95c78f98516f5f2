// assign_simt.cu -- register-tiled FP32 SIMT assignment kernel (small d).
//
// Assignment step, Eq. (3): rho_i = argmin_j ||x_i - c_j||,
// evaluated through the expansion ||x||^2 - 2 x.c + ||c||^2 (north_star):
// ||x_i||^2 is constant per row, so the kernel ranks the scores
//   s_ij = ||c_j||^2 + sum_k x_ik * (-2 c_jk)          (FFMA chain, fp32)
// and keeps, per row, the best score b1 (index i1, lowest index wins exact
// fp32 ties) and the runner-up score b2.  Rows whose computed gap b2 - b1 is
// within the rigorous fp32 error bound tau_i = gamma (||x_i||^2 + max||c||^2)
// are appended to the near-tie list and re-decided exactly in fp64 by
// refine.cu, so the labels equal the exact fp64 argmin.
//
// Layout: X row-major (n x d) fp32; each thread owns R rows held in
// registers; fl32(C) (pre-scaled by -2) and ||c||^2 are staged in shared memory in
// K-tiles and read as warp-broadcast vector loads.
#include "aakm_dev.cuh"

namespace aakm {

// Rigorous bound for the FFMA chain: each score has error
// <= (d+2) u (||x||^2 + 2 max||c||^2) for the chain, plus u (||x||^2 + ||c||^2)
// because the operand is fl32(c) of the fp64 centroid (2 |x.(c - fl32 c)| <=
// 2u ||x|| ||c||): (d+3) u (||x||^2 + 2 max||c||^2) per score, the gap of two
// scores twice that.  Flag when gap <= 2 * 2 (d+3) u (||x||^2 + cmax2) (factor
// 2 covers the 2 max||c||^2 term and ||x||^2 evaluated in fp32).
float tau_gamma_simt(int d) { return 8.0f * (float)(d + 3) * 5.9604645e-8f; }

template <int D>
struct RowsPerThread { static constexpr int value = D <= 4 ? 8 : (D <= 16 ? 4 : 2); };   // the most rows a thread keeps

__device__ __forceinline__ void push_flag(const Dev& d, int branch, bool flag, long long row, float b1, float tau) {
    unsigned mask = __ballot_sync(0xffffffffu, flag);
    if (mask == 0) return;
    int lane = threadIdx.x & 31;
    int leader = __ffs(mask) - 1;
    long long base = 0;
    if (lane == leader)
        base = (long long)atomicAdd((unsigned long long*)&d.flag_count[branch],
                                    (unsigned long long)__popc(mask));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (flag) {
        const long long f = base + __popc(mask & ((1u << lane) - 1));
        d.flag_rows[f] = (int)row;
        if (f < d.fcap) { d.flag_b1[f] = b1; d.flag_tau[f] = tau; }
    }
}

template <int D, int R>
__global__ void __launch_bounds__(256) k_assign_simt(Dev d, GEval g, int KT) {
    if (!geval_active(d, g)) return;
    extern __shared__ float4 smem4[];
    float* cs = reinterpret_cast<float*>(smem4);   // KT x D, holds -2 c
    float* cns = cs + KT * D;                      // KT
    int* lab_out = g.lab_out ? g.lab_out : d.lab[d.st->cur];
    const float cmax2 = __uint_as_float(d.st->cmax2_bits);

    float x[R][D];
    float b1[R], b2[R], xn[R];
    int i1[R];
    const long long row0 = (long long)blockIdx.x * (256 * R) + threadIdx.x;
    const bool al16 = ((uintptr_t)d.X & 15) == 0;   // X is borrowed: any float alignment works
#pragma unroll
    for (int r = 0; r < R; ++r) {
        long long row = row0 + (long long)r * 256;
        bool ok = row < d.n;
        float s = 0.f;
        if (D % 4 == 0 && al16) {                  // 16-B loads: a quarter of the load instructions
#pragma unroll
            for (int k = 0; k < D; k += 4) {
                const float4 v = ok ? __ldg(reinterpret_cast<const float4*>(d.X + row * D + k))
                                    : make_float4(0.f, 0.f, 0.f, 0.f);
                x[r][k] = v.x; x[r][k + 1] = v.y; x[r][k + 2] = v.z; x[r][k + 3] = v.w;
            }
        } else {
#pragma unroll
            for (int k = 0; k < D; ++k) x[r][k] = ok ? __ldg(d.X + row * D + k) : 0.f;
        }
#pragma unroll
        for (int k = 0; k < D; ++k) s = fmaf(x[r][k], x[r][k], s);
        xn[r] = s;
        b1[r] = INFINITY; b2[r] = INFINITY; i1[r] = 0;
    }

    for (int kt = 0; kt < d.K; kt += KT) {
        const int kc = min(KT, d.K - kt);
        __syncthreads();
        for (int e = threadIdx.x; e < kc * D; e += blockDim.x)
            cs[e] = -2.0f * d.C32[(long long)kt * D + e];
        for (int e = threadIdx.x; e < kc; e += blockDim.x) cns[e] = d.cn[kt + e];
        __syncthreads();
        // unrolled: the independent FFMA chains of four centroids interleave (one chain
        // of d dependent FFMAs per score would leave the pipe idle at 1 row per thread)
#pragma unroll 4
        for (int j = 0; j < kc; ++j) {
            float c[D];
            if constexpr (D % 4 == 0) {
#pragma unroll
                for (int k = 0; k < D; k += 4) {
                    float4 v = *reinterpret_cast<const float4*>(cs + j * D + k);
                    c[k] = v.x; c[k + 1] = v.y; c[k + 2] = v.z; c[k + 3] = v.w;
                }
            } else {
#pragma unroll
                for (int k = 0; k < D; ++k) c[k] = cs[j * D + k];
            }
            const float cnj = cns[j];
            const int jj = kt + j;
#pragma unroll
            for (int r = 0; r < R; ++r) {
                float s = cnj;
#pragma unroll
                for (int k = 0; k < D; ++k) s = fmaf(x[r][k], c[k], s);
                const bool p = s < b1[r];
                b2[r] = fminf(b2[r], fmaxf(s, b1[r]));
                i1[r] = p ? jj : i1[r];
                b1[r] = fminf(b1[r], s);
            }
        }
    }
    const float gam = d.tau_gamma;
#pragma unroll
    for (int r = 0; r < R; ++r) {
        long long row = row0 + (long long)r * 256;
        bool ok = row < d.n;
        const float tau = gam * (xn[r] + cmax2);
        bool flag = ok && (b2[r] - b1[r] <= tau);
        if (ok) lab_out[row] = i1[r];
        if (d.dbg_rows && ok) d.dbg_rows[row] = make_float4(b1[r], b2[r], tau, __int_as_float(i1[r]));
        push_flag(d, g.branch, flag, row, b1[r], tau);
    }
}

// Generic-d variant: the block's rows are staged transposed in shared memory
// (xs[k][tid]) so any d works; same scores, same tie/flag rules.
__global__ void __launch_bounds__(128) k_assign_simt_generic(Dev d, GEval g, int KT) {
    if (!geval_active(d, g)) return;
    extern __shared__ float4 smem4[];
    const int RB = blockDim.x;                       // rows per block (128, or 32 for large d)
    float* xs = reinterpret_cast<float*>(smem4);     // d x RB
    float* cs = xs + (size_t)d.d * RB;               // KT x d (-2c)
    float* cns = cs + (size_t)KT * d.d;              // KT
    int* lab_out = g.lab_out ? g.lab_out : d.lab[d.st->cur];
    const float cmax2 = __uint_as_float(d.st->cmax2_bits);
    const int D = d.d;
    const long long rbase = (long long)blockIdx.x * RB;
    for (int e = threadIdx.x; e < RB * D; e += RB) {
        int r = e / D, k = e % D;
        long long row = rbase + r;
        xs[k * RB + r] = row < d.n ? d.X[row * D + k] : 0.f;
    }
    __syncthreads();
    float xn = 0.f;
    for (int k = 0; k < D; ++k) xn = fmaf(xs[k * RB + threadIdx.x], xs[k * RB + threadIdx.x], xn);
    float b1 = INFINITY, b2 = INFINITY;
    int i1 = 0;
    for (int kt = 0; kt < d.K; kt += KT) {
        const int kc = min(KT, d.K - kt);
        __syncthreads();
        for (int e = threadIdx.x; e < kc * D; e += RB) cs[e] = -2.0f * d.C32[(long long)kt * D + e];
        for (int e = threadIdx.x; e < kc; e += RB) cns[e] = d.cn[kt + e];
        __syncthreads();
        for (int j = 0; j < kc; ++j) {
            float s = cns[j];
            const float* cj = cs + j * D;
            for (int k = 0; k < D; ++k) s = fmaf(xs[k * RB + threadIdx.x], cj[k], s);
            const bool p = s < b1;
            b2 = fminf(b2, fmaxf(s, b1));
            i1 = p ? kt + j : i1;
            b1 = fminf(b1, s);
        }
    }
    long long row = rbase + threadIdx.x;
    bool ok = row < d.n;
    const float tau = d.tau_gamma * (xn + cmax2);
    bool flag = ok && (b2 - b1 <= tau);
    if (ok) lab_out[row] = i1;
    if (d.dbg_rows && ok) d.dbg_rows[row] = make_float4(b1, b2, tau, __int_as_float(i1));
    push_flag(d, g.branch, flag, row, b1, tau);
}

template <int D, int R>
static void launch_r(const Dev& d, const GEval& g, cudaStream_t s) {
    int KT = d.K;
    const int max_smem = 96 * 1024;
    if ((size_t)KT * (D + 1) * 4 > (size_t)max_smem) KT = max_smem / ((D + 1) * 4);
    size_t smem = (size_t)KT * (D + 1) * 4;
    long long blocks = (d.n + 256LL * R - 1) / (256LL * R);
    if (blocks < 1) blocks = 1;
    k_assign_simt<D, R><<<(unsigned)blocks, 256, smem, s>>>(d, g, KT);
}

// Rows per thread: as many as RowsPerThread allows (register reuse of each C
// element) while the grid still covers every SM twice; small shards (c1: 10 000
// rows, c2: 100 000) drop to fewer rows per thread instead of leaving SMs idle.
template <int D>
static void launch_t(const Dev& d, const GEval& g, cudaStream_t s) {
    constexpr int RM = RowsPerThread<D>::value;
    const long long want = 2LL * d.num_sms * 256;                 // threads for two blocks per SM
    if (RM >= 8 && d.n >= want * 8) { launch_r<D, (RM >= 8 ? 8 : 1)>(d, g, s); return; }
    if (RM >= 4 && d.n >= want * 4) { launch_r<D, (RM >= 4 ? 4 : 1)>(d, g, s); return; }
    if (RM >= 2 && d.n >= want * 2) { launch_r<D, (RM >= 2 ? 2 : 1)>(d, g, s); return; }
    launch_r<D, 1>(d, g, s);
}

cudaError_t setup_simt() {
    cudaError_t e = cudaSuccess;
    auto set = [&](const void* f, int bytes) {
        cudaError_t r = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
        if (r != cudaSuccess) e = r;
    };
#define AAKM_SIMT_ATTR(D_)                                                  \
    set((const void*)k_assign_simt<D_, 1>, 96 * 1024);                      \
    set((const void*)k_assign_simt<D_, (RowsPerThread<D_>::value >= 2 ? 2 : 1)>, 96 * 1024); \
    set((const void*)k_assign_simt<D_, (RowsPerThread<D_>::value >= 4 ? 4 : 1)>, 96 * 1024); \
    set((const void*)k_assign_simt<D_, (RowsPerThread<D_>::value >= 8 ? 8 : 1)>, 96 * 1024);
    AAKM_SIMT_ATTR(1) AAKM_SIMT_ATTR(2) AAKM_SIMT_ATTR(3) AAKM_SIMT_ATTR(4) AAKM_SIMT_ATTR(8)
    AAKM_SIMT_ATTR(16) AAKM_SIMT_ATTR(32)
#undef AAKM_SIMT_ATTR
    set((const void*)k_assign_simt_generic, 200 * 1024);
    return e;
}

void launch_assign_simt(const Dev& d, const GEval& g, cudaStream_t s) {
    switch (d.d) {
        case 1: launch_t<1>(d, g, s); return;
        case 2: launch_t<2>(d, g, s); return;
        case 3: launch_t<3>(d, g, s); return;
        case 4: launch_t<4>(d, g, s); return;
        case 8: launch_t<8>(d, g, s); return;
        case 16: launch_t<16>(d, g, s); return;
        case 32: launch_t<32>(d, g, s); return;
        default: break;
    }
    const int max_smem = 200 * 1024;
    const int RB = d.d <= 256 ? 128 : 32;
    size_t xs = (size_t)d.d * RB * 4;
    long long KT = ((long long)max_smem - (long long)xs) / ((d.d + 1) * 4);
    if (KT > d.K) KT = d.K;
    if (KT < 1) KT = 1;
    size_t smem = xs + (size_t)KT * (d.d + 1) * 4;
    long long blocks = (d.n + RB - 1) / RB;
    if (blocks < 1) blocks = 1;
    k_assign_simt_generic<<<(unsigned)blocks, RB, smem, s>>>(d, g, (int)KT);
}

}  // namespace aakm
