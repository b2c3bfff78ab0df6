# K3 box limit: 4096 vs 65536 points (timing on the streams, decisions on the golden sets)
for m in 4096 65536; do
  SCUBA_OOB_ENUM_MAX=$m timeout 300 python tools/fast_sweep.py c3:100000 c4:100000 c5s:100000 2>&1 | grep ' ms ' | sed "s/^/max=$m: /"
  SCUBA_OOB_ENUM_MAX=$m timeout 300 python tools/enum_probe.py 2>&1 | grep -E 'crafted|random|corpus_m64' | sed "s/^/max=$m: /"
done
