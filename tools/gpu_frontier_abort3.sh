# frontier abort: factor x minimum grid (fast mode), then the C4 tail
for spec in "2 16" "1 4" "1 0" "2 4" "3 8"; do
  set -- $spec
  SCUBA_OOB_FRONTIER_ABORT=$1 SCUBA_OOB_FRONTIER_ABORT_MIN=$2 SCUBA_OOB_CHAIN=0 timeout 600 python tools/chain_ab.py c3:100000 c4:100000 2>&1 | grep chain= | cut -c1-120 | sed "s/^/fa=$1 min=$2 /"
done
python tools/tl_tail.py c4 100000 2>&1 | grep -v '^\[oob\]' | head -8
