# compute-sanitizer over every engine path (small batches), and the integer-pipe peaks with an in-kernel clock
mkdir -p gpurun_out
export CUDA_DEVICE_MAX_CONNECTIONS=32
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/alu_peak tools/alu_peak.cu && /tmp/alu_peak > gpurun_out/r02_alu_peak.jsonl; cat gpurun_out/r02_alu_peak.jsonl
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv,noheader >> gpurun_out/r02_alu_peak.jsonl
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_paths.py 300 > gpurun_out/r02_sanitizer_$tool.log 2>&1; echo "$tool rc=$?"; tail -4 gpurun_out/r02_sanitizer_$tool.log
done
