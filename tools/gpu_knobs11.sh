for rep in 1 2; do
for cfg in c3 c4 c5s; do
  run() { env "$@" timeout 600 python tools/knob_run.py $cfg 100000 "$LABEL" $HN >> gpurun_out/knobs11.txt 2>&1; }
  HN=0; LABEL=hn16; run X=1
  HN=24; LABEL=hn24; run X=1
  HN=32; LABEL=hn32; run X=1
done; done
grep -v "^\[" gpurun_out/knobs11.txt
