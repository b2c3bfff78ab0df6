# frontier speculative-lane abort: both modes (tools/fast_bench.py) at 0 / 1 / 2
for f in 0 1 2; do
  SCUBA_OOB_FRONTIER_ABORT=$f timeout 900 python tools/fast_bench.py c3:100000 c4:100000 2>&1 | grep -E 'n=' | cut -c1-120 | sed "s/^/fa=$f /"
done
