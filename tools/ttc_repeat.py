import sys, os
sys.path.insert(0, "/root/repo")
import torch
import bench
def barrier(): torch.cuda.synchronize()
for i in range(2):
    t = bench.time_to_converge("c4", 0, 1, barrier)
    print(i, t["iters"], t["dense_iters"], t["lloyd_iters"], t["energy"], t["lloyd_energy"], flush=True)
