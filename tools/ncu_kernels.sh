#!/bin/bash
# --set full on one launch of each kernel of interest (after the command ran clean without ncu)
TAG=${1:-r2}
ARGS="--steps 3 --warmup 2 --no-cpu --no-precompute --frames 0 --e2e-steps 0"
for K in k_local k_mplus_project k_vertex_pass k_energy_chunks k_hier_query_grp; do
  ncu --kernel-name regex:"$K" --launch-skip 2 --launch-count 1 --set full --import-source on --clock-control none \
      -o gpurun_out/${TAG}_full_$K python bench.py $ARGS > gpurun_out/${TAG}_ncu_$K.log 2>&1
  ncu -i gpurun_out/${TAG}_full_$K.ncu-rep --page details --csv > gpurun_out/${TAG}_c4_ncu_${K}.csv 2>/dev/null
  echo "$K $(grep -c . gpurun_out/${TAG}_c4_ncu_${K}.csv)"
  rm -f gpurun_out/${TAG}_full_$K.ncu-rep  # keep the CSV summary (gpurun_out returns <= 64 MiB)
done
