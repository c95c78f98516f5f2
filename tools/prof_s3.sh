set -x
python bench.py > gpurun_out/bench_s3.json 2> gpurun_out/bench_s3.err
bash tools/launches.sh c2 c3 c5
ncu --set full --clock-control none --import-source on -k regex:k_assign_tc -s 3 -c 1 -o gpurun_out/s3_c3_assign python tools/probe_tc.py auto 1000000 c3 > gpurun_out/ncu_c3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_assign_simt -s 3 -c 1 -o gpurun_out/s3_c2_assign python tools/probe_tc.py auto 100000 c2 > gpurun_out/ncu_c2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_assign_tc<2, 0" -s 2 -c 1 -o gpurun_out/s3_c5_assign python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 --ttc-config none --seed-config none > gpurun_out/ncu_c5.log 2>&1
ls gpurun_out
