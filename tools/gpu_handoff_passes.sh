# fast mode: hand-off to the frontier after N propagation passes (SCUBA_OOB_FAST_HEAVY_PASSES) A/B
for p in 128 384 1024 1000000; do
  SCUBA_OOB_FAST_HEAVY_PASSES=$p SCUBA_OOB_CHAIN=0 timeout 600 python tools/chain_ab.py c3:100000 c4:100000 c5s:100000 2>&1 | grep chain= | cut -c1-160 | sed "s/^/hp=$p /"
done
