# final r02 evidence of the current build: launch lists (c2-c5 bench runs) and ncu full
# captures of the c3 / c4 / c5 assignment kernels
bash tools/launches.sh c2 c3 c4 c5
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:k_assign_tc<.int.1, .int.0,' -s 2 -c 1 -o gpurun_out/s3_c3_assign python tools/probe_tc.py auto 1000000 c3 > gpurun_out/ncu_c3.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:k_assign_tc<.int.4, .int.0,' -s 2 -c 1 -o gpurun_out/s3_c4_assign python tools/probe_tc.py auto 4000000 c4 > gpurun_out/ncu_c4.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:k_assign_tc<.int.2, .int.0,' -s 2 -c 1 -o gpurun_out/s3_c5_assign python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 --ttc-config none --seed-config none > gpurun_out/ncu_c5.log 2>&1
