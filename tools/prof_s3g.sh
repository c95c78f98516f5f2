# final build: ncu full capture of the c4 assignment (four splitter warps), c4 launch list, smoke
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:k_assign_tc<.int.4, .int.0,' -s 2 -c 1 -o gpurun_out/s3g_c4_assign python tools/probe_tc.py auto 4000000 c4 > gpurun_out/ncu_c4g.log 2>&1
bash tools/launches.sh c4
python -c "import __graft_entry__ as g; g.smoke()"
