python -m pytest tests -m gpu -x -q -k "seed" 2>&1 | tail -1
for i in 1 2; do python bench.py --steps 1 --warmup 3 --e2e-steps 1 --ttc-config none --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); p=d['seed_pp']; print('c5 seed', round(p['seconds'],3), p['first_indices'])"; done
