#!/bin/bash
# Second half of the end-of-round measurement (compact outputs only; the .ncu-rep
# files stay on the box under /tmp and are summarised into gpurun_out/).
set -u
mkdir -p gpurun_out
timeout 900 python bench.py --config 3 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r01_bench_c3_final.log 2>&1; echo "bench3=$?"
timeout 600 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r01_bench_c4_final.log 2>&1; echo "bench4=$?"
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/plain_bench.log 2>&1 && \
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file /tmp/r01_bench_launches.csv $CMD > /tmp/ncu_bench.log 2>&1; echo "ncu_list=$?"
python tools/agg_launches.py /tmp/r01_bench_launches.csv 80 > gpurun_out/r01_bench_launches_summary.txt
gzip -c /tmp/r01_bench_launches.csv > gpurun_out/r01_bench_launches.csv.gz
for c in 2 3; do
  timeout 300 python tools/apply_probe.py --config $c --reps 3 > gpurun_out/plain_probe$c.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "probe/" \
    -k regex:k_apply -c 2 -o /tmp/r01_prof_apply_c$c python tools/apply_probe.py --config $c --reps 3 \
    > gpurun_out/ncu_full_c$c.log 2>&1; echo "ncu_full_c$c=$?"
  ncu -i /tmp/r01_prof_apply_c$c.ncu-rep --page raw --csv > gpurun_out/r01_prof_apply_c${c}_raw.csv 2>/dev/null
  ncu -i /tmp/r01_prof_apply_c$c.ncu-rep --page details --csv > gpurun_out/r01_prof_apply_c${c}_details.csv 2>/dev/null
done
timeout 1500 python bench.py --config 5 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r01_bench_c5_final.log 2>&1; echo "bench5=$?"
du -sh gpurun_out
