mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale_parity.py tests/test_gpu_partition.py tests/test_gpu_precompute.py -q -x -k "not contact_sweeps and not broadphase and not gauss_seidel_contact" > gpurun_out/ab_tests.log 2>&1; echo rc=$? >> gpurun_out/ab_tests.log
tail -3 gpurun_out/ab_tests.log
A="--steps 40 --warmup 3 --no-cpu --no-precompute --frames 0 --e2e-steps 0"
timeout 900 python bench.py $A > gpurun_out/ab_new.log 2>&1
JGS2_SPLIT_FWD=0 JGS2_SOLVE_FORK=0 JGS2_BWD_NARROW=0 timeout 900 python bench.py $A > gpurun_out/ab_old.log 2>&1
JGS2_BWD_NARROW=0 timeout 900 python bench.py $A > gpurun_out/ab_nonarrow.log 2>&1
JGS2_SOLVE_FORK=0 timeout 900 python bench.py $A > gpurun_out/ab_nofork.log 2>&1
for f in new old nonarrow nofork; do python - $f <<'P'
import json,sys
t=open(f"gpurun_out/ab_{sys.argv[1]}.log").read().strip().splitlines()
d=[json.loads(l) for l in t if l.startswith("{")]
if d: d=d[-1]; print(sys.argv[1], round(d["value"],2), d["phases_ms_per_step"]["factor_solve"], round(d["roofline"]["frac"],3))
else: print(sys.argv[1], t[-3:])
P
done
