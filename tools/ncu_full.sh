#!/bin/bash
# --set full of selected kernels over the C4 bench window; details exported as CSV (no .ncu-rep kept)
mkdir -p gpurun_out
TAG=$1; RE=$2; SKIP=${3:-10}; COUNT=${4:-4}
ARGS="--steps 4 --warmup 3 --no-cpu --no-precompute --frames 0 --e2e-steps 0"
ncu --kernel-name regex:"$RE" --launch-skip $SKIP --launch-count $COUNT --set full --import-source on \
    --clock-control none -o gpurun_out/${TAG} python bench.py $ARGS > gpurun_out/${TAG}.log 2>&1
ncu -i gpurun_out/${TAG}.ncu-rep --page details --csv > gpurun_out/${TAG}_details.csv 2>&1
rm -f gpurun_out/${TAG}.ncu-rep
python profiles/summarize_details.py gpurun_out/${TAG}_details.csv
