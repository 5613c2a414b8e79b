#!/bin/bash
# A/B of env settings on the short C4 bench: each argument is one variant ("-" = defaults)
mkdir -p gpurun_out
A="--steps 40 --warmup 3 --no-cpu --no-precompute --frames 0 --e2e-steps 0"
i=0
for v in "$@"; do
  i=$((i+1))
  if [ "$v" = "-" ]; then timeout 900 python bench.py $A > gpurun_out/abv_$i.log 2>&1
  else env $v timeout 900 python bench.py $A > gpurun_out/abv_$i.log 2>&1; fi
  python - gpurun_out/abv_$i.log "$v" <<'P'
import json,sys
t=open(sys.argv[1]).read().strip().splitlines()
d=[json.loads(l) for l in t if l.startswith("{")]
if d:
    d=d[-1]; ph=d["phases_ms_per_step"]
    print(f"{sys.argv[2]:50s} {d['value']:7.2f} sweeps/s  {d['ms_per_step']:6.2f} ms  solve {ph['factor_solve']:.3f} hess {ph['cubature_hessians']:.3f} local {ph['local_systems']:.3f}")
else: print(sys.argv[2], t[-3:])
P
done
