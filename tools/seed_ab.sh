# K-Means++ (all K centers): pruned D2 update vs the full pass, same indices
for c in c4 c3 c2; do for v in 1 0; do
  AAKM_SEED_PRUNE=$v python bench.py --config $c --steps 1 --warmup 3 --e2e-steps 1 --ttc-config none --no-cpu-baseline --seed-config $c 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); p=d['seed_pp']; print('$c prune=$v', round(p['seconds'],4), p['first_indices'], p['gpu_launches'])"
done; done
