// Standalone check of k_solve against a host Cholesky on a random window.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <vector>
#include "../../paper_1805_10638_b200/csrc/aa.cu"
using namespace aakm;
int main() {
    DevState* st; double* gp;
    cudaMalloc(&st, sizeof(DevState)); cudaMemset(st, 0, sizeof(DevState));
    cudaMalloc(&gp, AAKM_GRAM_BLOCKS * 2 * AAKM_H_SLOTS * 8);
    Dev d; memset(&d, 0, sizeof(d));
    const int H = 31, n = 40;
    d.st = st; d.gram_part = gp; d.H = H; d.m_max = 30; d.gram_blocks = 1; d.ridge = 1e-10;
    std::mt19937_64 rng(1);
    std::normal_distribution<double> nd;
    int fails = 0;
    for (int t : {1, 2, 3, 7, 29, 30, 31, 45}) for (int m : {0, 1, 3, 30}) {
        const int W = t < H - 1 ? t : H - 1;
        // dF(tau) random vectors for tau = t..t-W+1 ; F^t random
        std::vector<std::vector<double>> dF(W, std::vector<double>(n));
        std::vector<double> F(n);
        for (auto& v : dF) for (auto& x : v) x = nd(rng);
        if (W >= 3) dF[2] = dF[1];                               // duplicate column -> ridge / drop
        for (auto& x : F) x = nd(rng);
        DevState h; memset(&h, 0, sizeof(h));
        h.t = t; h.m = m; h.init_mode = 0;
        auto dot = [&](const std::vector<double>& a, const std::vector<double>& b) { double s = 0; for (int i = 0; i < n; ++i) s += a[i] * b[i]; return s; };
        for (int a = 1; a < W; ++a) for (int b = 1; b < W; ++b) h.gram[((t - a) % H) * H + (t - b) % H] = dot(dF[a], dF[b]);
        cudaMemcpy(st, &h, sizeof(h), cudaMemcpyHostToDevice);
        std::vector<double> part(2 * H, 0.0);
        for (int q = 0; q < W; ++q) { part[q] = dot(dF[0], dF[q]); part[W + q] = dot(dF[q], F); }
        cudaMemcpy(gp, part.data(), part.size() * 8, cudaMemcpyHostToDevice);
        k_solve<<<1, 32>>>(d);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("t=%d m=%d: %s\n", t, m, cudaGetErrorString(e)); return 1; }
        cudaMemcpy(&h, st, sizeof(h), cudaMemcpyDeviceToHost);
        int mt = std::min(m, W);
        // host: same rule (scaled normal eqs + ridge, drop oldest on failure)
        std::vector<double> th(mt, 0.0), s(mt);
        std::vector<int> act;
        for (int a = 0; a < mt; ++a) { s[a] = sqrt(dot(dF[a], dF[a])); if (s[a] > 0) act.push_back(a); }
        int na = act.size();
        while (na > 0) {
            std::vector<double> L(na * na, 0.0); bool ok = true;
            for (int i = 0; i < na && ok; ++i) for (int j = 0; j <= i; ++j) {
                double v = dot(dF[act[i]], dF[act[j]]) / (s[act[i]] * s[act[j]]) + (i == j ? 1e-10 : 0);
                for (int q = 0; q < j; ++q) v -= L[i * na + q] * L[j * na + q];
                if (i == j) { if (!(v > 0)) { ok = false; break; } L[i * na + i] = sqrt(v); } else L[i * na + j] = v / L[j * na + j];
            }
            if (!ok) { --na; continue; }
            std::vector<double> y(na);
            for (int i = 0; i < na; ++i) { double v = dot(dF[act[i]], F) / s[act[i]]; for (int q = 0; q < i; ++q) v -= L[i * na + q] * y[q]; y[i] = v / L[i * na + i]; }
            for (int i = na - 1; i >= 0; --i) { double v = y[i]; for (int q = i + 1; q < na; ++q) v -= L[q * na + i] * y[q]; y[i] = v / L[i * na + i]; }
            for (int i = 0; i < na; ++i) th[act[i]] = y[i] / s[act[i]];
            break;
        }
        double err = 0; for (int a = 0; a < mt; ++a) err = std::max(err, fabs(th[a] - h.theta[a]) / (1 + fabs(th[a])));
        double asum = 0; for (int j = 0; j < h.n_alpha; ++j) asum += h.alpha[j];
        bool good = h.m_t == mt && err < 1e-6 && fabs(asum - 1.0) < 1e-9;
        if (!good) ++fails;
        printf("t=%2d m=%2d m_t=%d n_alpha=%d max_theta_err=%.2e sum_alpha=%.12f %s\n", t, m, h.m_t, h.n_alpha, err, asum, good ? "ok" : "FAIL");
    }
    printf("fails=%d\n", fails);
    return fails != 0;
}
