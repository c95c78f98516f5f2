#!/bin/bash
# ncu launch list (time + DRAM bytes) of kmeans_seed_pp's kernels on c5 (12 centers)
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_seed -c 60 --csv \
    --log-file gpurun_out/seed_launches.csv python -c "
import torch
from paper_1805_10638_b200 import aakm, synthetic
X, _, c = synthetic.make('c5')
km = aakm.KMeans(torch.from_numpy(X).cuda(), 12, aakm.config())
km.seed_pp(synthetic.seed_uniforms('c5', 12))
km.close()" > gpurun_out/ncu_seed.log 2>&1
python tools/seed_shares.py gpurun_out/seed_launches.csv
