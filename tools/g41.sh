set -u
mkdir -p gpurun_out
timeout 1500 python bench.py --steps 3 --warmup 3 > gpurun_out/g41_b5.log 2>&1; echo "b5=$?"
timeout 600 python bench.py --config 2 --steps 10 --warmup 3 > gpurun_out/g41_b2.log 2>&1; echo b2=$?
timeout 900 python bench.py --config 3 --steps 3 --warmup 3 > gpurun_out/g41_b3.log 2>&1; echo b3=$?
timeout 600 python bench.py --config 4 --steps 5 --warmup 3 > gpurun_out/g41_b4.log 2>&1; echo b4=$?
timeout 600 python bench.py --config 1 --steps 10 --warmup 3 > gpurun_out/g41_b1.log 2>&1; echo b1=$?
for c in 2 3 4 5; do
  timeout 900 ncu --nvtx --nvtx-include "probe/" -k regex:k_apply --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/g41_apply_c$c.csv python tools/apply_probe.py --config $c --reps 2 > /dev/null 2>&1; echo "ncu_apply_c$c=$?"
done
timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "probe/" \
  -k regex:k_apply_orb2 -c 1 -f -o gpurun_out/g41_orb2_full python tools/apply_probe.py --config 5 --reps 1 --op smooth --steps 2 > gpurun_out/g41_ncu_orb2.log 2>&1; echo "ncu_full=$?"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/g41_bench_launches.csv \
   python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/g41_bench_ncu.log 2>&1; echo ncu=$?
python tools/agg_launches.py gpurun_out/g41_bench_launches.csv 60 > gpurun_out/g41_bench_launches_summary.txt
for b in 5 2 3 4 1; do tail -n 1 gpurun_out/g41_b$b.log | cut -c1-400; done
