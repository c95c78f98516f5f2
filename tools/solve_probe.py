"""k_solve phase clocks (AAKM_SOLVE_PROBE build, AAKM_TC_TRACE + AAKM_SOLVE_TRACE set):
P Algorithm 1 passes on CFG, then the last k_solve's clock64 stamps:
gram reduce, setup, factorization attempts, substitutions.  usage: solve_probe.py CFG P"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1805_10638_b200 import aakm, synthetic
cfg, P = sys.argv[1], int(sys.argv[2])
X, C0, c = synthetic.make(cfg, seed=0)
km = aakm.KMeans(torch.from_numpy(X).cuda(), c.K, aakm.config(m0=5))
km.aa_step(torch.from_numpy(C0).cuda(), info=False)
for _ in range(P):
    km.aa_step(info=False)
km.close()
v = [int(x) for x in open(os.environ["AAKM_SOLVE_TRACE"]).read().split()]
print(f"{cfg} after {P} passes: gram_reduce {v[1]-v[0]} clk, setup {v[2]-v[1]} clk, factor(all tries) {v[3]-v[2]} clk, "
      f"subst {v[4]-v[3]} clk, total {v[4]-v[0]} clk; tries {v[5]} na {v[6]} m_t {v[7]}")
