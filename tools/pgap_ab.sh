# pair-gap skip in the bounded engine: c4 bounded kmeans_run with and without (AAKM_NO_PGAP=1)
for r in 1 2; do for v in 0 1; do
  if [ $v = 1 ]; then export AAKM_NO_PGAP=1; else unset AAKM_NO_PGAP; fi
  echo "no_pgap=$v:"; python tools/run_timeline.py c4 bounded 2>&1 | grep -E " run: |k_refine_pair|k_bounds"
done; done
