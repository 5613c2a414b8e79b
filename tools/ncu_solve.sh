#!/bin/bash
# launch list of the factor-solve kernels over 2 timed sweeps (+ optional --set full of one kernel)
mkdir -p gpurun_out
TAG=${1:-solve}
ARGS="--steps 2 --warmup 3 --no-cpu --no-precompute --frames 0 --e2e-steps 0"
ncu --profile-from-start off --kernel-name regex:"apply|assemble|gather" \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active \
    --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py $ARGS > gpurun_out/${TAG}_list.log 2>&1
if [ -n "$2" ]; then
  ncu --kernel-name regex:"$2" --launch-skip ${3:-0} --launch-count 1 --set full --import-source on --clock-control none \
      -o gpurun_out/${TAG}_full python bench.py $ARGS > gpurun_out/${TAG}_full.log 2>&1
  ncu -i gpurun_out/${TAG}_full.ncu-rep --page details --csv > gpurun_out/${TAG}_full_details.csv 2>&1
  ncu -i gpurun_out/${TAG}_full.ncu-rep --page source --csv > gpurun_out/${TAG}_full_source.csv 2>&1
  rm -f gpurun_out/${TAG}_full.ncu-rep
fi
