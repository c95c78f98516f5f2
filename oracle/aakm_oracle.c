/*
 * aakm_oracle.c -- CPU ORACLE for Anderson-accelerated Lloyd K-Means
 * (arXiv 1805.10638).  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  The product path
 * (paper_1805_10638_b200/) never links, imports or executes it, and this file
 * shares no code, header, table or helper with the CUDA path.
 *
 * Plain, slow, obviously-correct: every quantity is computed in fp64 from its
 * definition in the paper, in the paper's order.  The samples X are fp32
 * values (BASELINE.json configs are fp32 data); everything derived from them
 * is fp64.  Floating-point contraction is disabled at build time
 * (-ffp-contract=off) so each sum is the literal left-to-right expression.
 * The only parallelism is an OpenMP loop over samples in the assignment step,
 * whose rows are independent (each row's arithmetic is identical to the
 * serial loop), so results do not depend on the thread count.
 *
 * Citations: PAPER.md:<line> of /root/reference/PAPER.md, and DESIGN.md
 * reading ids R-A1..R-A26 (= SURVEY.md §8c.3 A1..A26).
 *
 * Pins (tests/test_oracle_*.py, -m "not gpu"): SPEC/hand-derived worked
 * examples, the exact-rational Appendix-A trace (tests/golden/), brute-force
 * optimal partitions, scipy cdist argmin, numpy lstsq, sklearn Lloyd, and the
 * paper's invariants.  Every function below is pinned; none is "parity
 * unpinned".
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* Eq. (1)/(3) building block: squared Euclidean distance by DIRECT
 * differences (never the ||x||^2 - 2x.c + ||c||^2 expansion), summed over k in
 * ascending order.  PAPER.md:14 (Eq. 1), PAPER.md:30 (Eq. 3).                */
double ora_sqdist(const float *x, const double *c, int d)
{
    double acc = 0.0;
    for (int k = 0; k < d; ++k) {
        double diff = (double)x[k] - c[k];
        acc += diff * diff;
    }
    return acc;
}

/* Assignment step, Eq. (3) PAPER.md:28-32:
 *   rho_i = argmin_j ||x_i - c_j||.
 * Ties go to the lowest index (strict '<' while scanning j ascending) -- R-A16.
 * Labels are 0-based.                                                       */
void ora_assign(const float *X, int64_t N, int d, const double *C, int K,
                int32_t *labels)
{
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < N; ++i) {
        const float *x = X + i * (int64_t)d;
        double best = ora_sqdist(x, C, d);
        int32_t arg = 0;
        for (int j = 1; j < K; ++j) {
            double dj = ora_sqdist(x, C + (int64_t)j * d, d);
            if (dj < best) { best = dj; arg = j; }
        }
        labels[i] = arg;
    }
}

/* For tests: best and second-best fp64 distance of each row (the parity rule
 * needs the oracle's best-vs-chosen gap).                                    */
void ora_best2(const float *X, int64_t N, int d, const double *C, int K,
               double *best, double *second)
{
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < N; ++i) {
        const float *x = X + i * (int64_t)d;
        double b1 = INFINITY, b2 = INFINITY;
        for (int j = 0; j < K; ++j) {
            double dj = ora_sqdist(x, C + (int64_t)j * d, d);
            if (dj < b1) { b2 = b1; b1 = dj; }
            else if (dj < b2) { b2 = dj; }
        }
        best[i] = b1; second[i] = b2;
    }
}

/* Energy with a pre-computed assignment, E(P, C) -- Eq. (1) PAPER.md:14 and
 * Algorithm 1's E(P,.).  Summed in sample-index order.        */
double ora_energy(const float *X, int64_t N, int d, const double *C,
                  const int32_t *labels)
{
    double E = 0.0;
    for (int64_t i = 0; i < N; ++i)
        E += ora_sqdist(X + i * (int64_t)d, C + (int64_t)labels[i] * d, d);
    return E;
}

/* Update step, Eq. (4) PAPER.md:33-38:
 *   c_j = (1/N_j) sum_{i: rho_i = j} x_i,   N_j = #members.
 * Sums in sample-index order.  Empty cluster (N_j = 0, Eq. 4 undefined):
 * keep the row of C_prev, the centroids the assignment was made against
 * (R-A15).  counts may be NULL.                                             */
void ora_update(const float *X, int64_t N, int d, const int32_t *labels, int K,
                const double *C_prev, double *G, int64_t *counts)
{
    double *S = (double *)calloc((size_t)K * d, sizeof(double));
    int64_t *n = (int64_t *)calloc((size_t)K, sizeof(int64_t));
    for (int64_t i = 0; i < N; ++i) {
        int32_t j = labels[i];
        n[j] += 1;
        for (int k = 0; k < d; ++k)
            S[(int64_t)j * d + k] += (double)X[i * (int64_t)d + k];
    }
    for (int j = 0; j < K; ++j) {
        for (int k = 0; k < d; ++k) {
            int64_t o = (int64_t)j * d + k;
            G[o] = n[j] > 0 ? S[o] / (double)n[j] : C_prev[o];
        }
        if (counts) counts[j] = n[j];
    }
    free(S); free(n);
}

static double dot(const double *a, const double *b, int64_t n)
{
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s += a[i] * b[i];
    return s;
}

/* Least-squares problem of Eq. (7) PAPER.md:85-89 / Algorithm 1 PAPER.md:155:
 *   theta* = argmin || F^t - sum_j theta_j dF_j ||^2,
 *   dF_j = F^{t-j+1} - F^{t-j}, j = 1 (newest) .. m_t.
 * The paper does not state a solver (R-A14).  Reading R-A14, step by step:
 *   1. s_j = ||dF_j||; columns with s_j == 0 or non-finite are dropped;
 *   2. normal equations on unit-diagonal scaled columns:
 *        Gh_ab = <dF_a, dF_b>/(s_a s_b),  bh_a = <dF_a, F>/s_a;
 *   3. Cholesky of (Gh + ridge*I); if a pivot is <= 0 or non-finite, drop the
 *      oldest remaining column and retry; with no column left theta = 0;
 *   4. theta_j = phi_j / s_j (0 for dropped columns).
 * dF: m_t rows of length n (row j-1 is dF_j).  Returns the number of columns
 * finally used.                                                             */
int ora_ls_solve(const double *dF, const double *F, int64_t n, int m_t,
                 double ridge, double *theta)
{
    if (m_t <= 0) return 0;
    double *s = (double *)malloc(sizeof(double) * m_t);
    int *act = (int *)malloc(sizeof(int) * m_t);     /* active column ids   */
    double *L = (double *)malloc(sizeof(double) * m_t * m_t);
    double *Gh = (double *)malloc(sizeof(double) * m_t * m_t);
    double *bh = (double *)malloc(sizeof(double) * m_t);
    double *y = (double *)malloc(sizeof(double) * m_t);
    int na = 0;
    for (int j = 0; j < m_t; ++j) {
        theta[j] = 0.0;
        s[j] = sqrt(dot(dF + (int64_t)j * n, dF + (int64_t)j * n, n));
        if (s[j] > 0.0 && isfinite(s[j])) act[na++] = j;
    }
    for (int a = 0; a < m_t; ++a) {
        for (int b = 0; b < m_t; ++b) Gh[a * m_t + b] = 0.0;
        bh[a] = 0.0;
    }
    for (int a = 0; a < na; ++a) {
        int ja = act[a];
        bh[ja] = dot(dF + (int64_t)ja * n, F, n) / s[ja];
        for (int b = 0; b < na; ++b) {
            int jb = act[b];
            Gh[ja * m_t + jb] = dot(dF + (int64_t)ja * n, dF + (int64_t)jb * n, n)
                                / (s[ja] * s[jb]);
        }
    }
    int used = 0;
    while (na > 0) {
        /* Cholesky L L^T = Gh[act,act] + ridge I */
        int ok = 1;
        for (int a = 0; a < na && ok; ++a) {
            for (int b = 0; b <= a; ++b) {
                double v = Gh[act[a] * m_t + act[b]] + (a == b ? ridge : 0.0);
                for (int q = 0; q < b; ++q) v -= L[a * m_t + q] * L[b * m_t + q];
                if (a == b) {
                    if (!(v > 0.0) || !isfinite(v)) { ok = 0; break; }
                    L[a * m_t + a] = sqrt(v);
                } else {
                    L[a * m_t + b] = v / L[b * m_t + b];
                }
            }
        }
        if (!ok) { na -= 1; continue; }        /* act[] is newest-first: drop the oldest */
        for (int a = 0; a < na; ++a) {         /* forward: L y = bh */
            double v = bh[act[a]];
            for (int q = 0; q < a; ++q) v -= L[a * m_t + q] * y[q];
            y[a] = v / L[a * m_t + a];
        }
        for (int a = na - 1; a >= 0; --a) {    /* backward: L^T phi = y */
            double v = y[a];
            for (int q = a + 1; q < na; ++q) v -= L[q * m_t + a] * y[q];
            y[a] = v / L[a * m_t + a];
        }
        for (int a = 0; a < na; ++a) theta[act[a]] = y[a] / s[act[a]];
        used = na;
        break;
    }
    free(s); free(act); free(L); free(Gh); free(bh); free(y);
    return used;
}

/* Dynamic adjustment of m, Algorithm 1 PAPER.md:131-138 with constants from
 * PAPER.md:177.  Reading R-A5/R-A6: adjust only when the previous decrease
 * D = E^{t-2} - E^{t-1} is finite and > 0 (so t >= 3).  E_t is the candidate
 * (pre-guard) energy, E1/E2 the post-guard ones (R-A7).                     */
int ora_adjust_m(int m, int m_max, double E_t, double E1, double E2,
                 double eps1, double eps2)
{
    double D = E2 - E1;
    if (!(isfinite(D) && D > 0.0)) return m;
    double r = (E1 - E_t) / D;
    if (r < eps1) return m > 0 ? m - 1 : 0;
    if (r > eps2) return m < m_max ? m + 1 : m_max;
    return m;
}

/* ------------------------------------------------------------------------ */
/* Algorithm 1 as a state machine, one loop pass per call. */
typedef struct {
    /* problem */
    const float *X; int64_t N; int32_t d; int32_t K;
    /* config (PAPER.md:177 defaults; R-A18 m0) */
    int32_t m_max; double eps1; double eps2; int32_t dynamic_m;
    int64_t max_iters; double ridge;
    /* state */
    double *C;            /* C^t, K*d                                         */
    double *fallback;     /* C_AU^t = G^{t-1} (R-A3), K*d                     */
    double *Ghist;        /* (m_max+1) x K*d, row 0 = newest G               */
    double *Fhist;        /* (m_max+1) x K*d, row 0 = newest F               */
    int32_t hist_count;
    int32_t *labels_prev; /* P^{t-1}, N                                       */
    int32_t *labels;      /* scratch / result P, N                            */
    double E1, E2;        /* E^{t-1}, E^{t-2} (post-guard)                    */
    int32_t m;
    int32_t lloyd;        /* C^t is a plain Lloyd iterate (theta == 0)        */
    int64_t t;
    /* counters */
    int64_t n_accepted, n_rejected, n_assign;
    /* per-pass outputs (trace) */
    double E_cand, E_final; int64_t changed;
    int32_t m_t, rejected_now, accepted_now;
    double theta[64];
} ora_state;

static int64_t count_changed(const int32_t *a, const int32_t *b, int64_t N)
{
    int64_t c = 0;
    for (int64_t i = 0; i < N; ++i) c += (a[i] != b[i]);
    return c;
}

static void push_hist(ora_state *s, const double *G, const double *F)
{
    int64_t KD = (int64_t)s->K * s->d;
    int H = s->m_max + 1;
    int keep = s->hist_count < H ? s->hist_count : H - 1;
    memmove(s->Ghist + KD, s->Ghist, sizeof(double) * KD * keep);
    memmove(s->Fhist + KD, s->Fhist, sizeof(double) * KD * keep);
    memcpy(s->Ghist, G, sizeof(double) * KD);
    memcpy(s->Fhist, F, sizeof(double) * KD);
    s->hist_count = keep + 1;
}

/* Line 1 of Algorithm 1:
 *   C^1 = C_AU^1 = G(C^0);  F^0 = C^1 - C^0;  E^0 = +inf.
 * P^0 = Assign(C^0) (R-A4); the history holds (G^0, F^0); t = 1.           */
void ora_init(ora_state *s, const double *C0, int32_t m0)
{
    int64_t KD = (int64_t)s->K * s->d;
    double *G = (double *)malloc(sizeof(double) * KD);
    double *F = (double *)malloc(sizeof(double) * KD);
    ora_assign(s->X, s->N, s->d, C0, s->K, s->labels_prev);
    ora_update(s->X, s->N, s->d, s->labels_prev, s->K, C0, G, NULL);
    for (int64_t o = 0; o < KD; ++o) F[o] = G[o] - C0[o];
    s->hist_count = 0;
    push_hist(s, G, F);
    memcpy(s->C, G, sizeof(double) * KD);
    memcpy(s->fallback, G, sizeof(double) * KD);
    s->E1 = INFINITY; s->E2 = INFINITY;
    s->m = m0; s->lloyd = 1; s->t = 1;
    s->n_accepted = 0; s->n_rejected = 0; s->n_assign = 1;
    free(G); free(F);
}

/* One loop pass t of Algorithm 1 under reading R-A10
 * (rule R3).  Returns 0 = continue, 1 = converged (result in s->C,
 * s->labels, s->E_final), 2 = max_iters reached.                           */
int ora_pass(ora_state *s)
{
    int64_t KD = (int64_t)s->K * s->d;
    int64_t N = s->N;
    s->rejected_now = 0; s->accepted_now = 0; s->m_t = 0;
    for (int j = 0; j < 64; ++j) s->theta[j] = 0.0;

    /* PAPER.md:121  P^t = Assignment-Step(X, C^t);  PAPER.md:130 E^t = E(P^t, C^t) */
    ora_assign(s->X, N, s->d, s->C, s->K, s->labels);
    s->n_assign += 1;
    double E = ora_energy(s->X, N, s->d, s->C, s->labels);
    s->E_cand = E;
    s->changed = count_changed(s->labels, s->labels_prev, N);

    /* PAPER.md:122-125 convergence, rule R3: only a Lloyd iterate may stop */
    if (s->changed == 0 && s->lloyd) { s->E_final = E; return 1; }

    /* PAPER.md:131-138 dynamic m (candidate E^t, post-guard E^{t-1}, E^{t-2}) */
    if (s->dynamic_m)
        s->m = ora_adjust_m(s->m, s->m_max, E, s->E1, s->E2, s->eps1, s->eps2);

    /* PAPER.md:142-147 guard; R-A8 (>=), R-A9 (Lloyd iterates skip it),
     * R-A10 (an accelerated iterate repeating the partition is rejected)   */
    if (!s->lloyd) {
        if (E >= s->E1 || s->changed == 0) {
            memcpy(s->C, s->fallback, sizeof(double) * KD);
            ora_assign(s->X, N, s->d, s->C, s->K, s->labels);
            s->n_assign += 1;
            E = ora_energy(s->X, N, s->d, s->C, s->labels);
            s->n_rejected += 1; s->rejected_now = 1;
            s->lloyd = 1;
            s->changed = count_changed(s->labels, s->labels_prev, N);
            if (s->changed == 0) { s->E_final = E; return 1; }
        } else {
            s->n_accepted += 1; s->accepted_now = 1;
        }
    }
    s->E_final = E;

    /* PAPER.md:151-153  G^t = Update-Step(X, P^t); F^t = G^t - C^t */
    double *G = (double *)malloc(sizeof(double) * KD);
    double *F = (double *)malloc(sizeof(double) * KD);
    ora_update(s->X, N, s->d, s->labels, s->K, s->C, G, NULL);
    for (int64_t o = 0; o < KD; ++o) F[o] = G[o] - s->C[o];
    push_hist(s, G, F);   /* Ghist[j] = G^{t-j}, Fhist[j] = F^{t-j} */

    /* PAPER.md:154  m_t = min(m, t) */
    int m_t = s->m < s->t ? s->m : (int)s->t;
    if (m_t > s->hist_count - 1) m_t = s->hist_count - 1;
    s->m_t = m_t;
    double *Cn = (double *)malloc(sizeof(double) * KD);
    int all_zero = 1;
    if (m_t > 0) {
        /* PAPER.md:155 / Eq. (7): columns dF_j = F^{t-j+1} - F^{t-j} */
        double *dF = (double *)malloc(sizeof(double) * KD * m_t);
        for (int j = 1; j <= m_t; ++j)
            for (int64_t o = 0; o < KD; ++o)
                dF[(int64_t)(j - 1) * KD + o] =
                    s->Fhist[(int64_t)(j - 1) * KD + o] - s->Fhist[(int64_t)j * KD + o];
        ora_ls_solve(dF, s->Fhist, KD, m_t, s->ridge, s->theta);
        free(dF);
        for (int j = 0; j < m_t; ++j) if (s->theta[j] != 0.0) all_zero = 0;
    }
    /* PAPER.md:156  C^{t+1} = G^t - sum_j theta_j (G^{t-j+1} - G^{t-j})  (R-A1) */
    for (int64_t o = 0; o < KD; ++o) {
        double v = s->Ghist[o];
        for (int j = 1; j <= m_t; ++j)
            v -= s->theta[j - 1] *
                 (s->Ghist[(int64_t)(j - 1) * KD + o] - s->Ghist[(int64_t)j * KD + o]);
        Cn[o] = v;
    }
    s->lloyd = all_zero;

    /* bookkeeping for pass t+1 */
    memcpy(s->fallback, G, sizeof(double) * KD);   /* C_AU^{t+1} = G^t (R-A3) */
    memcpy(s->C, Cn, sizeof(double) * KD);
    s->E2 = s->E1; s->E1 = E;
    memcpy(s->labels_prev, s->labels, sizeof(int32_t) * N);
    s->t += 1;
    free(G); free(F); free(Cn);
    if (s->t > s->max_iters) return 2;
    return 0;
}

int ora_state_size(void) { return (int)sizeof(ora_state); }

/* ------------------------------------------------------------------------ */
/* K-Means++ seeding (the paper seeds with K-Means++ among others,
 * PAPER.md:44,347, citing Arthur & Vassilvitskii), with the
 * caller's uniforms u[0..k-1] in [0,1) and the D^2 weights in fixed point
 * (reading R-A27), step by step:
 *   t     = 50 - e with (2 max|x_ik|)^2 < 2^e: every squared coordinate
 *           difference scaled by 2^t is < 2^50;
 *   dist_i(c) = sum_k rint(((double)x_ik - (double)c_k)^2 * 2^t)   (int64,
 *           each term rounded to nearest-even; the sum is exact);
 *   center 0 = sample floor(u_0 N);  D2_i = dist_i(center 0);
 *   for r = 1..k-1:  M = max_i D2_i (M = 0: fewer than k distinct samples ->
 *           return 2);  sh = max(0, bitlen(M) + ceil(log2 N) - 62);
 *           w_i = D2_i >> sh;  T = sum_i w_i;  tau = min(T - 1, floor(u_r T));
 *           center r = the smallest i with w_0 + ... + w_i > tau  (inverse CDF:
 *           P(i) = w_i / T, proportional to D^2; w_i = 0 is never drawn);
 *           D2_i = min(D2_i, dist_i(center r)).
 * idx[k] receives the sample indices; D2_out (optional, N) the final D2.
 * Returns 0, 1 (a u outside [0,1) or k outside [1, N]) or 2.               */
static int64_t ora_q(double v, int t) { return (int64_t)nearbyint(ldexp(v, t)); }

static int64_t ora_qdist(const float *x, const float *c, int d, int t)
{
    int64_t s = 0;
    for (int k = 0; k < d; ++k) {
        double diff = (double)x[k] - (double)c[k];
        s += ora_q(diff * diff, t);
    }
    return s;
}

int ora_seed_pp(const float *X, int64_t N, int d, int k, const double *u,
                int64_t *idx, int64_t *D2_out)
{
    if (k < 1 || (int64_t)k > N) return 1;
    for (int r = 0; r < k; ++r)
        if (!(u[r] >= 0.0 && u[r] < 1.0)) return 1;
    double amax = 0.0;
    for (int64_t i = 0; i < N * (int64_t)d; ++i)
        if (fabs((double)X[i]) > amax) amax = fabs((double)X[i]);
    int e = 0;
    if (amax > 0.0) frexp(4.0 * amax * amax, &e);       /* (2 amax)^2 < 2^e */
    const int t = 50 - e;
    int L = 0;
    while (((int64_t)1 << L) < N) ++L;                  /* ceil(log2 N) */
    int64_t *D2 = (int64_t *)malloc((size_t)N * sizeof(int64_t));
    int64_t i0 = (int64_t)floor(u[0] * (double)N);
    if (i0 > N - 1) i0 = N - 1;
    idx[0] = i0;
    for (int64_t i = 0; i < N; ++i)
        D2[i] = ora_qdist(X + i * (int64_t)d, X + i0 * (int64_t)d, d, t);
    int status = 0;
    for (int r = 1; r < k; ++r) {
        int64_t M = 0;
        for (int64_t i = 0; i < N; ++i)
            if (D2[i] > M) M = D2[i];
        if (M == 0) { status = 2; break; }
        int bl = 0;
        while (bl < 63 && (M >> bl) != 0) ++bl;         /* M < 2^bl */
        int sh = bl + L - 62;
        if (sh < 0) sh = 0;
        int64_t T = 0;
        for (int64_t i = 0; i < N; ++i) T += D2[i] >> sh;
        int64_t tau = (int64_t)floor(u[r] * (double)T);
        if (tau > T - 1) tau = T - 1;
        int64_t acc = 0, pick = -1;
        for (int64_t i = 0; i < N; ++i) {
            acc += D2[i] >> sh;
            if (acc > tau) { pick = i; break; }
        }
        idx[r] = pick;
        for (int64_t i = 0; i < N; ++i) {
            int64_t v = ora_qdist(X + i * (int64_t)d, X + pick * (int64_t)d, d, t);
            if (v < D2[i]) D2[i] = v;
        }
    }
    if (D2_out) memcpy(D2_out, D2, (size_t)N * sizeof(int64_t));
    free(D2);
    return status;
}
