// aa.cu -- the Anderson step and the device-side control of Algorithm 1
// (PAPER.md:107-160), replicated on every rank from allreduced scalars.
//
//   k_control   convergence rule R3 (R-A10), dynamic m
//               (R-A5..A7), energy guard (PAPER.md:142-147,
//               R-A8, R-A9): writes the device predicates reject / done.
//   k_finalize  G^t = Update-Step (Eq. 4; G = S/N, empty -> C row,
//               R-A15), F^t = G^t - C^t into ring slot t%H.
//   k_gram      <dF(t), dF(tau)> and <dF(tau), F^t> for the window (Eq. 7 /
//               PAPER.md:155; "m inner products between (Kd)-dimensional
//               vectors"); fixed-grid fp64 partials.
//   k_solve     fixed-order reduction of the partials, column-scaled ridge
//               Cholesky with drop-oldest (R-A14) -> theta -> mixing weights.
//   k_combine   C^{t+1} = G^t - sum_j theta_j (G^{t-j+1} - G^{t-j})
//               (minus sign R-A1) = sum_j alpha_j G^{t-j},
//               fused with the centroid prep of the next assignment (fl32(C),
//               ||c||^2, max ||c||^2; the tensor operands follow in k_csplit16/32).
//   k_advance   E^{t-2} <- E^{t-1} <- E^t, P^{t-1} <- P^t, t <- t+1, trace.
// All reductions are fixed-order, so every rank computes identical bytes.
#include <math.h>

#include "aakm_dev.cuh"

namespace aakm {

// ---------------------------------------------------------------- combine
// mode 0: mix from (st->alpha, st->alpha_slot, st->n_alpha), active if !done
// mode 1: C <- G[st->fb_slot] (fallback C_AU^t = G^{t-1}, R-A3), active if reject
// mode 2: C <- src (caller centroids / C^0), always
// C^t is fp64 (the whole Anderson state is, R-A17); fl32(C) for SIMT and ||c||^2
// are derived from it here, the tensor engines' operands by k_csplit16 / k_csplit32.
__global__ void __launch_bounds__(256) k_combine(Dev d, int mode, const double* src) {
    DevState* st = d.st;
    if (mode == 0 && st->done) return;
    if (mode == 1 && (st->done || !st->reject)) return;
    const int D = d.d;
    const long long KD = (long long)d.K * D;
    const int lane = threadIdx.x & 31;
    const long long w0 = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const long long nw = (long long)gridDim.x * (blockDim.x >> 5);
    int na = 1;
    double al[AAKM_H_SLOTS];
    const double* base[AAKM_H_SLOTS];
    if (mode == 0) {
        na = st->n_alpha;
        for (int q = 0; q < na; ++q) { al[q] = st->alpha[q]; base[q] = d.Gring + (long long)st->alpha_slot[q] * KD; }
    } else if (mode == 1) {
        al[0] = 1.0; base[0] = d.Gring + (long long)st->fb_slot * KD;
    } else {
        al[0] = 1.0; base[0] = src;
    }
    float bmax = 0.f;
    for (long long j = w0; j < d.K; j += nw) {
        double nrm = 0.0;
        for (int k = lane; k < D; k += 32) {
            const long long e = j * D + k;
            double c;
            if (na == 1 && al[0] == 1.0) {
                c = base[0][e];
            } else {
                c = 0.0;
                for (int q = 0; q < na; ++q) c = fma(al[q], base[q][e], c);   // C^{t+1} = sum_j alpha_j G^{t-j}
            }
            d.C[e] = c;
            if (d.C32) d.C32[e] = (float)c;
            nrm = fma(c, c, nrm);
        }
        for (int o = 16; o; o >>= 1) nrm += __shfl_xor_sync(0xffffffffu, nrm, o);
        const float cnj = (float)nrm;
        if (lane == 0) d.cn[j] = cnj;
        bmax = fmaxf(bmax, __double2float_ru(nrm));
    }
    // max ||c||^2: per-block max -> atomicMax into cmax2_tmp; last block publishes and resets
    for (int o = 16; o; o >>= 1) bmax = fmaxf(bmax, __shfl_xor_sync(0xffffffffu, bmax, o));
    __shared__ float wm[32];
    __shared__ bool last;
    if (lane == 0) wm[threadIdx.x >> 5] = bmax;
    __syncthreads();
    if (threadIdx.x == 0) {
        float m = 0.f;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) m = fmaxf(m, wm[i]);
        atomicMax(&st->cmax2_tmp, __float_as_uint(m));      // non-negative floats order as uints
        __threadfence();
        last = atomicAdd(&st->comb_ctr, 1u) == gridDim.x - 1;
        if (last) {
            __threadfence();
            st->cmax2_bits = atomicExch(&st->cmax2_tmp, 0u);
            st->comb_ctr = 0;
        }
    }
}

void launch_combine(const Dev& d, int mode, const double* src, cudaStream_t s) {
    long long warps = d.K;
    int blocks = (int)((warps + 7) / 8);
    if (blocks > 1184) blocks = 1184;
    if (blocks < 1) blocks = 1;
    k_combine<<<blocks, 256, 0, s>>>(d, mode, src);
}

// ---------------------------------------------------------------- control
__device__ int adjust_m(int m, int m_max, double Et, double E1, double E2, double eps1, double eps2) {
    // PAPER.md:131-138; R-A5/R-A6: only with a finite, positive previous decrease
    const double D = E2 - E1;
    if (!(isfinite(D) && D > 0.0)) return m;
    const double r = (E1 - Et) / D;
    if (r < eps1) return m > 0 ? m - 1 : 0;
    if (r > eps2) return m < m_max ? m + 1 : m_max;
    return m;
}

__global__ void k_control(Dev d, int stage) {
    DevState* st = d.st;
    if (st->done) return;
    if (stage == 1 && !st->reject) return;
    {
        // E = (E_hi + 2^-30 E_lo) / q from the reduced fixed-point parts (what k_energy
        // does for the API calls), fused here: one single-thread launch per G-evaluation
        long long* pk = d.packed[stage];
        const double q = energy_q(d);
        const long long* e = pk + pk_ehi(d);
        pk[pk_e(d)] = __double_as_longlong(((double)e[0] + (double)e[1] * 9.313225746154785e-10) / q);
    }
    if (stage == 0) {
        const long long* pk = d.packed[0];
        const double E = __longlong_as_double(pk[pk_e(d)]);   // k_energy, after the allreduce
        const long long ch = pk[pk_ch(d)];
        st->n_assign += 1;
        st->last_flag[0] = d.flag_count[0];
        st->rows_total += d.n;
        st->rows_scored += (d.ub && st->bnd_use) ? d.act_count[0] : d.n;
        st->reject = 0; st->accepted_now = 0; st->rejected_now = 0;
        st->E_cand = E; st->E_final = E; st->changed = ch;
        if (st->init_mode) return;                              // line 1: E^0 = +inf regardless
        if (ch == 0 && st->lloyd) {                             // PAPER.md:122-125, rule R3
            st->done = 1; st->converged = 1;
            return;
        }
        if (d.dynamic_m) st->m = adjust_m(st->m, d.m_max, E, st->E1, st->E2, d.eps1, d.eps2);
        if (!st->lloyd) {                                       // R-A9: Lloyd iterates skip the guard
            if (E >= st->E1 || ch == 0) {                       // PAPER.md:142 (>=, R-A8); R-A10
                st->reject = 1; st->rejected_now = 1; st->n_rejected += 1;
                st->fb_slot = (int)((st->t - 1) % d.H);         // C_AU^t = G^{t-1} (R-A3)
                if (d.condB) cudaGraphSetConditional(d.condB, 1u);   // graph replay: run branch B
            } else {
                st->accepted_now = 1; st->n_accepted += 1;
            }
        }
    } else {
        if (!st->reject) return;
        const long long* pk = d.packed[1];
        const double E = __longlong_as_double(pk[pk_e(d)]);
        const long long ch = pk[pk_ch(d)];
        st->n_assign += 1;
        st->last_flag[1] = d.flag_count[1];
        st->rows_total += d.n;
        st->rows_scored += (d.ub && st->bnd_use) ? d.act_count[1] : d.n;
        st->E_final = E; st->changed = ch;
        st->lloyd = 1;
        if (ch == 0) { st->done = 1; st->converged = 1; }       // R3: re-test after the fallback
    }
}

void launch_control(const Dev& d, int stage, cudaStream_t s) { k_control<<<1, 1, 0, s>>>(d, stage); }

// ---------------------------------------------------------------- finalize
__global__ void __launch_bounds__(256) k_finalize(Dev d) {
    DevState* st = d.st;
    if (st->done) return;
    const int D = d.d;
    const long long KD = (long long)d.K * D;
    const long long* pk = st->reject ? d.packed[1] : d.packed[0];
    const long long slot = st->t % d.H;
    double* G = d.Gring + slot * KD;
    double* F = d.Fring + slot * KD;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < KD;
         e += (long long)gridDim.x * blockDim.x) {
        const long long nj = pk[pk_n(d) + e / D];
        const double c = d.C[e];
        const double g = nj > 0 ? fx_value(pk[e], pk[KD + e], d.fx_inv) / (double)nj : c;   // G = S / N (Eq. 4)
        G[e] = g;
        F[e] = g - c;                                            // F^t = G^t - C^t (fp64)
        if (d.sref) {                                            // S(P^t), N(P^t): the next pass's S_ref
            d.sref[e] = pk[e];
            d.sref[KD + e] = pk[KD + e];
        }
    }
    if (d.sref) {
        for (long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x; j < d.K; j += (long long)gridDim.x * blockDim.x)
            d.sref[2 * KD + j] = pk[pk_n(d) + j];
        if (blockIdx.x == 0 && threadIdx.x == 0) st->sref_valid = 1;
    }
}

void launch_finalize(const Dev& d, cudaStream_t s) {
    long long KD = (long long)d.K * d.d;
    int blocks = (int)((KD + 255) / 256);
    if (blocks > 1184) blocks = 1184;
    k_finalize<<<blocks, 256, 0, s>>>(d);
}

// ---------------------------------------------------------------- gram
// For the window tau = t, t-1, ..., t-W+1 (W = min(t, H-1)):
//   q < W : <dF(t), dF(t-q)>,   q >= W : <dF(t-(q-W)), F^t>,
// dF(tau) = F^tau - F^{tau-1} formed in fp64 from the fp64 ring.
__global__ void __launch_bounds__(128) k_gram(Dev d) {
    DevState* st = d.st;
    if (st->done || st->init_mode) return;
    const long long t = st->t;
    const int H = d.H;
    const int W = (int)(t < H - 1 ? t : H - 1);
    const long long KD = (long long)d.K * d.d;
    double acc_g[AAKM_H_SLOTS - 1], acc_b[AAKM_H_SLOTS - 1];
#pragma unroll
    for (int q = 0; q < AAKM_H_SLOTS - 1; ++q) { acc_g[q] = 0.0; acc_b[q] = 0.0; }
    const double* F[AAKM_H_SLOTS];
    for (int q = 0; q <= W; ++q) F[q] = d.Fring + ((t - q) % H) * KD;   // F^{t-q}
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < KD;
         e += (long long)gridDim.x * blockDim.x) {
        const double ft = F[0][e];
        double prev = ft;
        double dft = 0.0;
#pragma unroll
        for (int q = 0; q < AAKM_H_SLOTS - 1; ++q) {
            if (q < W) {
                const double older = F[q + 1][e];
                const double df = prev - older;                  // dF(t-q)
                if (q == 0) dft = df;
                acc_g[q] = fma(dft, df, acc_g[q]);
                acc_b[q] = fma(df, ft, acc_b[q]);
                prev = older;
            }
        }
    }
    __shared__ __align__(16) double red[4][2 * (AAKM_H_SLOTS - 1)];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int q = 0; q < W; ++q) {
        double a = acc_g[q], b = acc_b[q];
        for (int o = 16; o; o >>= 1) {
            a += __shfl_xor_sync(0xffffffffu, a, o);
            b += __shfl_xor_sync(0xffffffffu, b, o);
        }
        if (lane == 0) { red[w][q] = a; red[w][W + q] = b; }
    }
    __syncthreads();
    for (int q = threadIdx.x; q < 2 * W; q += blockDim.x) {
        double v = 0.0;
        for (int i = 0; i < 4; ++i) v += red[i][q];
        d.gram_part[(long long)blockIdx.x * 2 * H + q] = v;
    }
}

void launch_gram(const Dev& d, cudaStream_t s) { k_gram<<<d.gram_blocks, 128, 0, s>>>(d); }

// ---------------------------------------------------------------- solve
// One warp.  Eq. (7) under reading R-A14 (see oracle ora_ls_solve for the
// plain statement): unit-diagonal scaling, ridge, Cholesky, drop-oldest.
// Lane r owns row r of the matrix / Cholesky factor in shared memory.
#define FULL 0xffffffffu
// Fixed-order reduction of this pass's Gram partials: one warp per entry, lanes
// stride over the blocks, then a fixed xor tree (same bytes on every rank).
__device__ __forceinline__ void gram_reduce(const Dev& d) {
    DevState* st = d.st;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int H = d.H;
    const long long t = st->t;
    const int init = st->init_mode;
    const int W = init ? 0 : (int)(t < H - 1 ? t : H - 1);
    const int ts = (int)(t % H);
    for (int q = warp; q < 2 * W; q += 32) {
        double v = 0.0;
        for (int b = lane; b < d.gram_blocks; b += 32) v += d.gram_part[(long long)b * 2 * H + q];
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) {
            if (q < W) {
                const int s2 = (int)((t - q) % H);
                st->gram[ts * H + s2] = v;
                st->gram[s2 * H + ts] = v;
            } else {
                st->bvec[q - W] = v;
            }
        }
    }
}

// one block: all 32 warps reduce the Gram partials (fixed order), then warp 0 solves
__global__ void __launch_bounds__(1024) k_solve(Dev d) {
    DevState* st = d.st;
    if (st->done) return;
    gram_reduce(d);
    __syncthreads();                                 // st->gram / st->bvec written by the block
    if (threadIdx.x >= 32) return;
    const int lane = threadIdx.x;
    const int H = d.H;
    const long long t = st->t;
    const int init = st->init_mode;
    const int W = init ? 0 : (int)(t < H - 1 ? t : H - 1);
    const int ts = (int)(t % H);
    int m_t = init ? 0 : (st->m < t ? st->m : (int)t);
    if (m_t > W) m_t = W;
    // column a <-> dF(t - a); lane a holds column a's scale and rhs
    const int sa = (int)((((t - lane) % H) + H) % H);
    double s_a = 0.0, b_a = 0.0;
    bool act = false;
    if (lane < m_t) {
        s_a = sqrt(st->gram[sa * H + sa]);
        act = s_a > 0.0 && isfinite(s_a);
        b_a = act ? st->bvec[lane] / s_a : 0.0;
    }
    // compact the active columns (newest first): lane i <- column idx[i]
    const unsigned am = __ballot_sync(FULL, act);
    int na = __popc(am);
    int col = -1;                                   // column held by this lane after compaction
    {
        // the i-th set bit of am
        unsigned m = am;
        for (int i = 0; i < lane && m; ++i) m &= m - 1;
        col = (lane < na) ? __ffs(m) - 1 : -1;
    }
    const int my_slot = col >= 0 ? (int)((((t - col) % H) + H) % H) : 0;
    const double my_s = __shfl_sync(FULL, s_a, col >= 0 ? col : 0);
    const double my_b = __shfl_sync(FULL, b_a, col >= 0 ? col : 0);
    // The compacted, scaled, ridged normal matrix in shared memory (lane i = row i):
    // all loads issued at once, then a right-looking Cholesky in which each lane
    // updates its own row.  Every entry sees the same subtraction sequence as the
    // dot-product form (q ascending), so theta is unchanged bit for bit.
    __shared__ double sA[AAKM_H_SLOTS][AAKM_H_SLOTS + 1];    // scaled matrix (kept for restarts)
    __shared__ double sL[AAKM_H_SLOTS][AAKM_H_SLOTS + 1];    // factor, built in place
    __shared__ double s_s[AAKM_H_SLOTS];
    __shared__ int s_slot[AAKM_H_SLOTS];
    if (lane < na) { s_slot[lane] = my_slot; s_s[lane] = my_s; }
    __syncwarp();
    if (lane < na) {
        for (int c = 0; c <= lane; ++c) sA[lane][c] = st->gram[my_slot * H + s_slot[c]];
        for (int c = 0; c <= lane; ++c) sA[lane][c] = sA[lane][c] / (my_s * s_s[c]) + (c == lane ? d.ridge : 0.0);
    }
    __syncwarp();
    double phi_mine = 0.0;
    while (na > 0) {
        if (lane < na)
            for (int c = 0; c <= lane; ++c) sL[lane][c] = sA[lane][c];
        __syncwarp();
        bool ok = true;
        for (int c = 0; c < na; ++c) {
            const double diag = sL[c][c];
            if (!(diag > 0.0) || !isfinite(diag)) { ok = false; break; }
            const double Lcc = sqrt(diag);
            double Lic = 0.0;
            if (lane > c && lane < na) { Lic = sL[lane][c] / Lcc; sL[lane][c] = Lic; }
            __syncwarp();
            if (lane == c) sL[c][c] = Lcc;
            if (lane > c && lane < na)
                for (int j = c + 1; j <= lane; ++j) sL[lane][j] -= Lic * sL[j][c];
            __syncwarp();
        }
        if (!ok) { --na; __syncwarp(); continue; }   // drop the oldest active column
        // forward: L y = bh (lane a ends up holding y_a)
        double y_mine = 0.0;
        double bres = my_b;                          // b_i - sum_{q < a} L_iq y_q, q ascending
        for (int a = 0; a < na; ++a) {
            const double ya = __shfl_sync(FULL, bres, a) / sL[a][a];
            if (lane == a) y_mine = ya;
            if (lane > a && lane < na) bres -= sL[lane][a] * ya;
        }
        // backward: L^T phi = y (fixed xor-tree sums)
        phi_mine = 0.0;
        for (int a = na - 1; a >= 0; --a) {
            double contrib = (lane > a && lane < na) ? sL[lane][a] * phi_mine : 0.0;
            for (int o = 16; o; o >>= 1) contrib += __shfl_xor_sync(FULL, contrib, o);
            const double ya = __shfl_sync(FULL, y_mine, a);
            const double pa = (ya - contrib) / sL[a][a];
            if (lane == a) phi_mine = pa;
        }
        break;
    }
    // theta per original column: theta_col = phi / s
    double th_lane = 0.0;                            // theta of column `lane`
    {
        const double th_c = (col >= 0 && col < m_t && lane < na) ? phi_mine / my_s : 0.0;
        // scatter back: column j takes th_c from the lane holding it
        for (int i = 0; i < AAKM_H_SLOTS; ++i) {
            const int ci = __shfl_sync(FULL, (lane < na) ? col : -1, i);
            const double v = __shfl_sync(FULL, th_c, i);
            if (ci == lane) th_lane = v;
        }
    }
    const unsigned nz = __ballot_sync(FULL, lane < m_t && th_lane != 0.0);
    // alpha_0 = 1 - theta_1, alpha_j = theta_j - theta_{j+1}, alpha_{m_t} = theta_{m_t}
    const double th_prev = __shfl_up_sync(FULL, th_lane, 1);     // theta of column lane-1
    if (lane < m_t) st->theta[lane] = th_lane;
    if (lane <= m_t) {
        const double tj = lane >= 1 ? th_prev : 1.0;              // "theta_0" := 1
        const double tj1 = lane < m_t ? th_lane : 0.0;
        st->alpha[lane] = tj - tj1;
        st->alpha_slot[lane] = (int)((((t - lane) % H) + H) % H);
    }
    __syncwarp();
    if (lane == 0) {
        const int allzero = nz == 0;
        st->m_t = m_t;
        st->n_alpha = allzero ? 1 : m_t + 1;
        if (allzero) { st->alpha[0] = 1.0; st->alpha_slot[0] = ts; }
        st->lloyd = allzero;
    }
}
#undef FULL

void launch_solve(const Dev& d, cudaStream_t s) { k_solve<<<1, 1024, 0, s>>>(d); }

// ---------------------------------------------------------------- advance
__global__ void k_advance(Dev d) {
    DevState* st = d.st;
    if (st->done) {
        if (!st->final_traced) {
            st->final_traced = 1;
            if (!st->init_mode && st->trace_len < AAKM_TRACE_CAP) {
                TraceRec r;
                r.t = st->t; r.changed = st->changed; r.E_cand = st->E_cand; r.E_final = st->E_final;
                r.m = st->m; r.m_t = 0; r.accepted = 0; r.rejected = st->rejected_now;
                r.converged = st->converged; r.lloyd = 1;
                d.trace[st->trace_len++] = r;
            }
        }
        return;
    }
    if (st->init_mode) {                                   // end of Algorithm 1 line 1
        st->init_mode = 0; st->t = 1; st->m = d.m0; st->lloyd = 1;
        st->E1 = INFINITY; st->E2 = INFINITY;              // E^0 = +inf
        st->hist_count = 1; st->cur ^= 1;
        return;
    }
    if (st->trace_len < AAKM_TRACE_CAP) {
        TraceRec r;
        r.t = st->t; r.changed = st->changed; r.E_cand = st->E_cand; r.E_final = st->E_final;
        r.m = st->m; r.m_t = st->m_t; r.accepted = st->accepted_now; r.rejected = st->rejected_now;
        r.converged = 0; r.lloyd = st->lloyd;
        d.trace[st->trace_len++] = r;
    }
    st->E2 = st->E1; st->E1 = st->E_final;
    st->hist_count = st->hist_count + 1 < d.H ? st->hist_count + 1 : d.H;
    st->t += 1;
    if (st->t > d.max_iters) {
        // stop (not converged) with C = C^{t+1} and the labels P^t of the pass just
        // run; cur is NOT flipped, so lab[cur] holds P^t as after a converged stop
        st->done = 1; st->converged = 0; st->final_traced = 1;
        return;
    }
    st->cur ^= 1;
}

void launch_advance(const Dev& d, cudaStream_t s) { k_advance<<<1, 1, 0, s>>>(d); }

__global__ void k_reset(Dev d) {
    DevState* st = d.st;
    st->t = 0; st->n_accepted = 0; st->n_rejected = 0; st->n_assign = 0; st->changed = 0;
    st->last_flag[0] = st->last_flag[1] = 0; st->trace_len = 0;
    st->E1 = INFINITY; st->E2 = INFINITY; st->E_cand = 0.0; st->E_final = 0.0;
    st->m = d.m0; st->m_t = 0; st->lloyd = 1; st->reject = 0;
    st->done = 0; st->converged = 0; st->init_mode = 1;
    st->hist_count = 0; st->accepted_now = 0; st->rejected_now = 0; st->label_error = 0;
    st->n_alpha = 1; st->fb_slot = 0; st->final_traced = 0;
    st->bnd_ready = 0; st->bnd_use = 0;                         // bounded engine: recompute every row first
    st->sref_valid = 0; st->use_delta = 0;                      // incremental update: no S(P^{t-1}) yet
    st->n_upd = 0; st->n_delta = 0; st->rows_moved = 0;
    st->rows_scored = 0; st->rows_total = 0;
}

void launch_reset(const Dev& d, cudaStream_t s) { k_reset<<<1, 1, 0, s>>>(d); }

}  // namespace aakm
