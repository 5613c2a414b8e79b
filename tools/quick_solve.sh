#!/bin/bash
# solve-touching GPU tests + one short bench (new build), optional env A/B as $1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale_parity.py tests/test_gpu_partition.py tests/test_gpu_precompute.py -q -x -k "not contact_sweeps and not broadphase and not gauss_seidel_contact" > gpurun_out/q_tests.log 2>&1; echo rc=$? >> gpurun_out/q_tests.log
tail -2 gpurun_out/q_tests.log
A="--steps 40 --warmup 3 --no-cpu --no-precompute --frames 0 --e2e-steps 0"
timeout 900 python bench.py $A > gpurun_out/q_bench.log 2>&1
[ -n "$1" ] && env $1 timeout 900 python bench.py $A > gpurun_out/q_bench_b.log 2>&1
for f in q_bench q_bench_b; do [ -f gpurun_out/$f.log ] && python - gpurun_out/$f.log <<'P'
import json,sys
t=open(sys.argv[1]).read().strip().splitlines()
d=[json.loads(l) for l in t if l.startswith("{")]
if d: d=d[-1]; print(sys.argv[1], round(d["value"],2), d["phases_ms_per_step"], round(d["roofline"]["frac"],3))
else: print(sys.argv[1], t[-3:])
P
done
