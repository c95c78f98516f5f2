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
    pdl_wait();                                     // PDL: the predecessor's writes are visible
    pdl_trigger();
    DevState* st = d.st;
    if (mode == 0 && st->done) return;
    if (mode == 1 && (st->done || !st->reject)) return;
    const int D = d.d;
    const long long KD = (long long)d.K * D;
    const int lane = threadIdx.x & 31;
    const long long w0 = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const long long nw = (long long)gridDim.x * (blockDim.x >> 5);
    // mixing weights and their ring rows in shared memory (a runtime-indexed local
    // array would live in local memory)
    __shared__ double al[AAKM_H_SLOTS];
    __shared__ const double* base[AAKM_H_SLOTS];
    const int na = mode == 0 ? st->n_alpha : 1;
    if (threadIdx.x < (unsigned)na) {
        if (mode == 0) {
            al[threadIdx.x] = st->alpha[threadIdx.x];
            base[threadIdx.x] = d.Gring + (long long)st->alpha_slot[threadIdx.x] * KD;
        } else {
            al[0] = 1.0;
            base[0] = mode == 1 ? d.Gring + (long long)st->fb_slot * KD : src;
        }
    }
    __syncthreads();
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
    launch_pdl(k_combine, blocks, 256, 0, s, d, mode, src);
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
    pdl_wait();                                     // PDL: the predecessor's writes are visible
    pdl_trigger();
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

void launch_control(const Dev& d, int stage, cudaStream_t s) { launch_pdl(k_control, 1, 1, 0, s, d, stage); }

// ---------------------------------------------------------------- finalize
__global__ void __launch_bounds__(256) k_finalize(Dev d) {
    pdl_wait();                                     // PDL: the predecessor's writes are visible
    pdl_trigger();
    DevState* st = d.st;
    if (st->done) return;
    const int D = d.d;
    const long long KD = (long long)d.K * D;
    const long long* pk = st->reject ? d.packed[1] : d.packed[0];
    const long long* pl = st->reject ? d.partial[1] : d.partial[0];   // this rank's own sums (S_ref)
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
        if (d.sref) {                                            // S(P^t), N(P^t) of this rank: the next S_ref
            d.sref[e] = pl[e];
            d.sref[KD + e] = pl[KD + e];
        }
    }
    if (d.sref) {
        for (long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x; j < d.K; j += (long long)gridDim.x * blockDim.x)
            d.sref[2 * KD + j] = pl[pk_n(d) + j];
        if (blockIdx.x == 0 && threadIdx.x == 0) st->sref_valid = 1;
    }
}

void launch_finalize(const Dev& d, cudaStream_t s) {
    long long KD = (long long)d.K * d.d;
    int blocks = (int)((KD + 255) / 256);
    if (blocks > 1184) blocks = 1184;
    launch_pdl(k_finalize, blocks, 256, 0, s, d);
}

// ---------------------------------------------------------------- gram
// For the window tau = t, t-1, ..., t-W+1 (W = min(t, H-1)):
//   q < W : <dF(t), dF(t-q)>,   q >= W : <dF(t-(q-W)), F^t>,
// dF(tau) = F^tau - F^{tau-1} formed in fp64 from the fp64 ring.
__global__ void __launch_bounds__(128) k_gram(Dev d) {
    pdl_wait();                                     // PDL: the predecessor's writes are visible
    pdl_trigger();
    DevState* st = d.st;
    if (st->done || st->init_mode) return;
    const long long t = st->t;
    const int H = d.H;
    const int W = (int)(t < H - 1 ? t : H - 1);
    const long long KD = (long long)d.K * d.d;
    constexpr int Q = AAKM_H_SLOTS - 1;
    // ring offsets of F^{t-q} in shared memory, the window loops fully unrolled with a
    // (block-uniform) predicate: the accumulators stay in registers (a runtime-indexed
    // array went to local memory) and the W + 1 ring loads of an element issue together
    __shared__ long long soff[AAKM_H_SLOTS];
    if (threadIdx.x <= W) soff[threadIdx.x] = ((t - threadIdx.x) % H) * KD;
    __syncthreads();
    double acc_g[Q], acc_b[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) { acc_g[q] = 0.0; acc_b[q] = 0.0; }
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < KD;
         e += (long long)gridDim.x * blockDim.x) {
        const double ft = d.Fring[soff[0] + e];
        double prev = ft;
        double dft = 0.0;
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            if (q < W) {
                const double older = d.Fring[soff[q + 1] + e];
                const double df = prev - older;                  // dF(t-q)
                if (q == 0) dft = df;
                acc_g[q] = fma(dft, df, acc_g[q]);
                acc_b[q] = fma(df, ft, acc_b[q]);
                prev = older;
            }
        }
    }
    __shared__ __align__(16) double red[4][2 * Q];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        if (q < W) {
            double a = acc_g[q], b = acc_b[q];
#pragma unroll
            for (int o = 16; o; o >>= 1) {
                a += __shfl_xor_sync(0xffffffffu, a, o);
                b += __shfl_xor_sync(0xffffffffu, b, o);
            }
            if (lane == 0) { red[w][q] = a; red[w][W + q] = b; }
        }
    }
    __syncthreads();
    for (int q = threadIdx.x; q < 2 * W; q += blockDim.x) {
        double v = 0.0;
        for (int i = 0; i < 4; ++i) v += red[i][q];
        d.gram_part[(long long)blockIdx.x * 2 * H + q] = v;
    }
}

void launch_gram(const Dev& d, cudaStream_t s) { launch_pdl(k_gram, d.gram_blocks, 128, 0, s, d); }

// ---------------------------------------------------------------- solve
// One warp.  Eq. (7) under reading R-A14 (see oracle ora_ls_solve for the
// plain statement): unit-diagonal scaling, ridge, Cholesky, drop-oldest.
// Lane r owns row r of the matrix / Cholesky factor in shared memory.
#define FULL 0xffffffffu
// AAKM_SOLVE_PROBE builds: clock64 phase stamps of the last k_solve (perf only)
#ifdef AAKM_SOLVE_PROBE
#define SOLVE_STAMP(i) do { if (d.dbg_ts && threadIdx.x == 0) d.dbg_ts[2 * 8 * 256 + (i)] = clock64(); } while (0)
#else
#define SOLVE_STAMP(i) do { } while (0)
#endif
// Fixed-order reduction of this pass's Gram partials: one warp per entry, lanes
// stride over the blocks, then a fixed xor tree (same bytes on every rank).
__device__ __forceinline__ void gram_reduce(const Dev& d) {
    DevState* st = d.st;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (int)(blockDim.x >> 5);
    const int H = d.H;
    const long long t = st->t;
    const int init = st->init_mode;
    const int W = init ? 0 : (int)(t < H - 1 ? t : H - 1);
    const int ts = (int)(t % H);
    // entry q = warp + u * nw (u < EPW) of warp `warp`; every load of a lane in flight
    // at once (blocks b = lane + 32 bb), then a fixed xor tree per entry
    constexpr int EPW = 4, BPL = (AAKM_GRAM_BLOCKS + 31) / 32;
    double v[EPW];
#pragma unroll
    for (int u = 0; u < EPW; ++u) v[u] = 0.0;
#pragma unroll
    for (int bb = 0; bb < BPL; ++bb) {
        const int b = lane + 32 * bb;
#pragma unroll
        for (int u = 0; u < EPW; ++u) {
            const int q = warp + u * nw;
            if (b < d.gram_blocks && q < 2 * W) v[u] += d.gram_part[(long long)b * 2 * H + q];
        }
    }
#pragma unroll
    for (int u = 0; u < EPW; ++u) {
        const int q = warp + u * nw;
        double x = v[u];
#pragma unroll
        for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        if (lane == 0 && q < 2 * W) {
            if (q < W) {
                const int s2 = (int)((t - q) % H);
                st->gram[ts * H + s2] = x;
                st->gram[s2 * H + ts] = x;
            } else {
                st->bvec[q - W] = x;
            }
        }
    }
}

// One block of 512 threads: its 16 warps reduce the Gram partials (fixed order);
// warp 0 scales and compacts the columns; one thread per lower-triangle entry
// factors the scaled, ridged normal matrix (right-looking Cholesky, the entry in
// a register, two block barriers per column); warp 0 substitutes.  The
// arithmetic is the oracle's (ora_ls_solve: sqrt, correctly rounded divisions,
// no contraction; every factor entry and forward-substitution value subtracts
// its terms in the same ascending order); only the back substitution subtracts
// in descending order (right-looking: a serial ascending chain per row costs
// more than the rest of the solve).  The Gram itself is a fixed-grid sum here,
// a serial dot there, so theta agrees to rounding, not bitwise.
constexpr int SOLVE_THREADS = 512;
static_assert((AAKM_H_SLOTS - 1) * AAKM_H_SLOTS / 2 <= SOLVE_THREADS, "one thread per entry (m_t <= H - 1)");
static_assert(2 * (AAKM_H_SLOTS - 1) <= 4 * (SOLVE_THREADS / 32), "gram_reduce: EPW entries per warp");
__global__ void __launch_bounds__(SOLVE_THREADS) k_solve(Dev d) {
    pdl_wait();                                     // PDL: the predecessor's writes are visible
    pdl_trigger();
    DevState* st = d.st;
    if (st->done) return;
    SOLVE_STAMP(0);
    gram_reduce(d);
    __syncthreads();                                 // st->gram / st->bvec written by the block
    SOLVE_STAMP(1);
    const int tid = threadIdx.x, lane = tid & 31;
    const int H = d.H;
    const long long t = st->t;
    const int init = st->init_mode;
    const int W = init ? 0 : (int)(t < H - 1 ? t : H - 1);
    const int ts = (int)(t % H);
    int m_t = init ? 0 : (st->m < t ? st->m : (int)t);
    if (m_t > W) m_t = W;
    __shared__ double sL[AAKM_H_SLOTS][AAKM_H_SLOTS + 1];    // the factor (written once at the end)
    __shared__ double s_s[AAKM_H_SLOTS], s_b[AAKM_H_SLOTS];
    __shared__ double colv[AAKM_H_SLOTS], sdiag[AAKM_H_SLOTS];
    __shared__ int s_slot[AAKM_H_SLOTS], s_col[AAKM_H_SLOTS];
    __shared__ int s_na, s_ok;
    if (tid < 32) {
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
        const int na = __popc(am);
        unsigned m = am;
        for (int i = 0; i < lane && m; ++i) m &= m - 1;          // the lane-th set bit of am
        const int col = (lane < na) ? __ffs(m) - 1 : -1;
        const double my_s = __shfl_sync(FULL, s_a, col >= 0 ? col : 0);
        const double my_b = __shfl_sync(FULL, b_a, col >= 0 ? col : 0);
        if (lane < na) {
            s_slot[lane] = (int)((((t - col) % H) + H) % H);
            s_s[lane] = my_s; s_b[lane] = my_b; s_col[lane] = col;
        }
        if (lane == 0) s_na = na;
    }
    __syncthreads();
    int na = s_na;
    // this thread's entry (ei, ej), ej <= ei: tid = ei (ei + 1) / 2 + ej
    int ei = 0;
    while ((ei + 1) * (ei + 2) / 2 <= tid) ++ei;
    const int ej = tid - ei * (ei + 1) / 2;
    double a0 = 0.0;                                 // the scaled, ridged entry (kept for restarts)
    if (ei < na)
        a0 = __dadd_rn(__ddiv_rn(st->gram[s_slot[ei] * H + s_slot[ej]], __dmul_rn(s_s[ei], s_s[ej])), ei == ej ? d.ridge : 0.0);
    double phi_mine = 0.0;
    SOLVE_STAMP(2);
    int tries = 0;
    while (na > 0) {
        ++tries;
        const bool act = ei < na;
        double a = a0;
        bool ok = true;
        for (int c = 0; c < na; ++c) {
            if (act && ei == c && ej == c) {         // pivot (its trailing updates are done)
                const bool okc = a > 0.0 && isfinite(a);
                s_ok = okc;
                a = okc ? sqrt(a) : 0.0;             // L_cc
                sdiag[c] = a;
            }
            __syncthreads();
            if (!s_ok) { ok = false; break; }
            if (act && ej == c && ei > c) { a = __ddiv_rn(a, sdiag[c]); colv[ei] = a; }   // L_ic
            __syncthreads();
            if (act && ej > c) a = __dsub_rn(a, __dmul_rn(colv[ei], colv[ej]));       // trailing update
        }
        SOLVE_STAMP(3);
        if (!ok) { --na; __syncthreads(); continue; }   // drop the oldest active column
        if (act) sL[ei][ej] = a;
        __syncthreads();
        if (tid < 32) {
            // forward: L y = bh, y_a = (bh_a - sum_{q < a, ascending} L_aq y_q) / L_aa
            double y_mine = 0.0;
            double bres = lane < na ? s_b[lane] : 0.0;
            for (int q = 0; q < na; ++q) {
                const double yq = __ddiv_rn(__shfl_sync(FULL, bres, q), sdiag[q]);
                if (lane == q) y_mine = yq;
                if (lane > q && lane < na) bres = __dsub_rn(bres, __dmul_rn(sL[lane][q], yq));
            }
            // backward: L^T phi = y, right-looking: phi_a = (y_a - sum_{q > a} L_qa phi_q) / L_aa
            // with the q terms subtracted as the phi_q appear (descending q; the oracle's
            // dot-product form subtracts them ascending -- the one ordering difference)
            double res = y_mine;
            for (int q = na - 1; q >= 0; --q) {
                const double pq = __ddiv_rn(__shfl_sync(FULL, res, q), sdiag[q]);
                if (lane == q) phi_mine = pq;
                if (lane < q) res = __dsub_rn(res, __dmul_rn(sL[q][lane], pq));
            }
        }
        break;
    }
    SOLVE_STAMP(4);
#ifdef AAKM_SOLVE_PROBE
    if (d.dbg_ts && tid == 0) { d.dbg_ts[2 * 8 * 256 + 5] = tries; d.dbg_ts[2 * 8 * 256 + 6] = na; d.dbg_ts[2 * 8 * 256 + 7] = m_t; }
#endif
    (void)tries;
    if (tid >= 32) return;
    const int col = lane < na ? s_col[lane] : -1;
    const double my_s = lane < na ? s_s[lane] : 1.0;
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

void launch_solve(const Dev& d, cudaStream_t s) { launch_pdl(k_solve, 1, SOLVE_THREADS, 0, s, d); }

// ---------------------------------------------------------------- advance
__global__ void k_advance(Dev d) {
    pdl_wait();                                     // PDL: the predecessor's writes are visible
    pdl_trigger();
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

void launch_advance(const Dev& d, cudaStream_t s) { launch_pdl(k_advance, 1, 1, 0, s, d); }

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
