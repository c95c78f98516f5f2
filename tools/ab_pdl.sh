# A/B of programmatic dependent launch (AAKM_PDL=0/1) on whole kmeans_run passes
for r in 1 2; do for v in 0 1; do
  for c in c1 c2 c3; do echo -n "PDL=$v "; AAKM_PDL=$v python tools/run_timeline.py $c 2>/dev/null | head -1; done
done; done
