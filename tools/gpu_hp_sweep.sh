# fast mode: pass-based hand-off threshold around the default (two repeats each)
for p in 128 96 64 48 128 96 64 48; do
  SCUBA_OOB_FAST_HEAVY_PASSES=$p timeout 300 python tools/fast_sweep.py c3:100000 c4:100000 2>&1 | grep ' ms ' | sed "s/^/hp=$p: /"
done
