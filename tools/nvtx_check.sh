# NVTX ranges: ncu restricted to one Algorithm 1 step's range (eager aa_step passes on c2)
ncu --nvtx --nvtx-include "aakm:assign/" --metrics gpu__time_duration.sum --csv --log-file gpurun_out/nvtx_assign.csv \
  python tools/per_config.py c2 2 1 > gpurun_out/nvtx_run.log 2>&1
ncu --nvtx --nvtx-include "aakm:anderson/" --metrics gpu__time_duration.sum --csv --log-file gpurun_out/nvtx_anderson.csv \
  python tools/per_config.py c2 2 1 >> gpurun_out/nvtx_run.log 2>&1
python tools/shares.py gpurun_out/nvtx_assign.csv gpurun_out/nvtx_anderson.csv
