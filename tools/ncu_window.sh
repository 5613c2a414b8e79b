#!/bin/bash
# ncu launch list (duration + DRAM bytes per launch) over K sweeps after W warm-up sweeps of the
# C4 bench (steady state: the balls resting on the floor), all kernels.
mkdir -p gpurun_out
TAG=${1:-win}; W=${2:-100}; K=${3:-3}
ARGS="--steps $K --warmup $W --no-cpu --no-precompute --frames 0 --e2e-steps 0"
ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py $ARGS > gpurun_out/${TAG}_list.log 2>&1
python profiles/parse_launches.py gpurun_out/${TAG}_launches.csv > gpurun_out/${TAG}_summary.txt
head -40 gpurun_out/${TAG}_summary.txt
