#!/bin/bash
# ncu evidence for profiles/ (run on the GPU box, after the same command exited 0 without ncu):
#  1. launch list over the bench's timed window (cudaProfilerStart/Stop around it), per-launch
#     duration + DRAM bytes (cold-cache, serialised: shares, not absolutes)
#  2. --set full on the top kernels (one launch each)
set -e
mkdir -p gpurun_out
TAG=${1:-r2}
ARGS="--steps 4 --warmup 3 --no-cpu --no-precompute --frames 0 --e2e-steps 0"
ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py $ARGS > gpurun_out/${TAG}_ncu_list.log 2>&1
python profiles/parse_launches.py gpurun_out/${TAG}_launches.csv > gpurun_out/${TAG}_c4_launches.txt
head -25 gpurun_out/${TAG}_c4_launches.txt
ncu --kernel-name regex:"${NCU_FULL_RE:-k_fwd_apply$|k_local|k_mplus_project|k_vertex_pass}" \
    --launch-skip ${NCU_FULL_SKIP:-20} --launch-count ${NCU_FULL_COUNT:-4} \
    --set full --import-source on --clock-control none -o gpurun_out/${TAG}_full python bench.py $ARGS \
    > gpurun_out/${TAG}_ncu_full.log 2>&1
tail -2 gpurun_out/${TAG}_ncu_full.log
# per-kernel details as CSV (the .ncu-rep stays out of gpurun_out: 64 MiB cap)
ncu -i gpurun_out/${TAG}_full.ncu-rep --page details --csv > gpurun_out/${TAG}_full_details.csv 2>&1 || true
rm -f gpurun_out/${TAG}_full.ncu-rep
