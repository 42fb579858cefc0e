#!/bin/bash
# A/B of solver variants on the bench workload: prints ms/step and phase times
run() { name=$1; shift; env "$@" python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab_$name.log 2>&1;
  python -c "import json; d=json.loads(open('gpurun_out/ab_$name.log').read().strip().splitlines()[-1]); print('$name', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['phases_ms'].items()}, d['iters'], d['gpu_launches'])"; }
for v in "$@"; do run ${v%%:*} ${v#*:}; done
