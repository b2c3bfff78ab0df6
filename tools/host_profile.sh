# Sampling profile of the host pipeline (SCUBA_OOB_PROF, host.cpp): runs
# tools/host_profile.py without a CUDA context and writes the library-relative
# program counters to gpurun_out/host_prof.txt; symbolize with
#   python tools/agg_prof.py gpurun_out/host_prof.txt
# usage: bash tools/host_profile.sh [cfg] [iterations]
mkdir -p gpurun_out
CUDA_VISIBLE_DEVICES= SCUBA_OOB_PROF=gpurun_out/host_prof.txt python tools/host_profile.py ${1:-c3} ${2:-100}
tail -1 gpurun_out/host_prof.txt
