mkdir -p gpurun_out
for c in 32 8 16; do
  for i in 1 2; do CUDA_DEVICE_MAX_CONNECTIONS=$c timeout 300 python tools/corpus_wall.py fast --cold-only 2>&1 | tail -1 | sed "s/^/conn=$c cold: /"; done
  CUDA_DEVICE_MAX_CONNECTIONS=$c SCUBA_OOB_CHAIN=0 timeout 600 python tools/chain_ab.py c3:100000 c4:100000 2>&1 | grep chain= | cut -c1-140 | sed "s/^/conn=$c /"
done
