#!/bin/bash
# usage: tools/quick.sh TAG  -- GPU tests + short bench lines for the main paths/configs into gpurun_out/
T=${1:-q}
python -m pytest tests -m gpu -x -q > gpurun_out/${T}_pytest.log 2>&1; tail -3 gpurun_out/${T}_pytest.log
for a in "c5 auto" "c5 tc" "c4 auto" "c3 auto"; do set -- $a
  python bench.py --config $1 --path $2 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/${T}_bench_$1_$2.json 2> gpurun_out/${T}_bench_$1_$2.err
  python -c "import json,sys; l=json.load(open(sys.argv[1])); r=l['roofline']; print(sys.argv[1], l['config']['assign_path'], 'ms/step %.2f'%l['ms_per_step'], 'assign_ms %.2f'%r['avg_launch_ms'], 'frac %.3f'%r['frac'], 'value %.3e'%l['value'])" gpurun_out/${T}_bench_$1_$2.json || tail -5 gpurun_out/${T}_bench_$1_$2.err
done
