for c in c4 c5 c4 c5; do python tools/probe_tc.py auto 4000000 $c 2>&1 | grep -v Warn; done
python -m pytest tests -m gpu -x -q 2>&1 | tail -3
