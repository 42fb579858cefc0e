#!/bin/bash
# End-of-round measurement on one B200 (run under gpurun from the repo root):
# GPU test suite, smoke, bench lines for configs 2-5, the bench launch list and
# ncu full captures of the fine-level apply passes.  Outputs in gpurun_out/.
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r01_pytest_gpu_final.log 2>&1; echo "pytest=$?"
tail -3 gpurun_out/r01_pytest_gpu_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r01_smoke_final.log 2>&1; echo "smoke=$?"
timeout 600 python bench.py > gpurun_out/r01_bench_c2_final.log 2>&1; echo "bench=$?"
tail -1 gpurun_out/r01_bench_c2_final.log
timeout 900 python bench.py --config 3 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r01_bench_c3_final.log 2>&1; echo "bench3=$?"
timeout 600 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r01_bench_c4_final.log 2>&1; echo "bench4=$?"
timeout 900 python bench.py --config 5 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r01_bench_c5_final.log 2>&1; echo "bench5=$?"
tail -1 gpurun_out/r01_bench_c5_final.log | cut -c1-400
# launch list of the bench command (cold-cache, serialised: compare shares)
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/plain_bench.log 2>&1 && \
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r01_bench_launches.csv $CMD > gpurun_out/ncu_bench.log 2>&1; echo "ncu_list=$?"
# full capture of the fine apply (both colour passes) at configs 2 and 3
for c in 2 3; do
  timeout 300 python tools/apply_probe.py --config $c --reps 3 > gpurun_out/plain_probe$c.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "probe/" \
    -k regex:k_apply -c 2 -o gpurun_out/r01_prof_apply_c$c python tools/apply_probe.py --config $c --reps 3 \
    > gpurun_out/ncu_full_c$c.log 2>&1; echo "ncu_full_c$c=$?"
done
