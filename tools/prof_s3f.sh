python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for c in c4 c5; do python tools/probe_tc.py auto 4000000 $c 2>&1 | grep -v Warn; done
for v in 2 4 2 4; do echo -n "NSW=$v "; AAKM_TC_NSW=$v python tools/probe_tc.py auto 4000000 c3 2>&1 | grep -v Warn; done
python tools/per_config.py c4 2>&1 | grep -v Warn | cut -c1-260
python bench.py --steps 3 --warmup 3 --e2e-steps 1 --seed-config none --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); t=d['time_to_converge']; print('ttc', t['seconds'], t['iters'], t['lloyd_seconds'], t['dense_seconds'])"
