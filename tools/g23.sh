set -u
mkdir -p gpurun_out
timeout 1500 python bench.py --steps 3 --warmup 2 > gpurun_out/g23_bench.log 2>&1; echo "bench=$?"
tail -c 4000 gpurun_out/g23_bench.log
timeout 900 ncu --nvtx --nvtx-include "probe/" -k regex:k_apply --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/g23_apply_c5.csv python tools/apply_probe.py --config 5 --reps 2 > gpurun_out/g23_apply_ncu.log 2>&1; echo "ncu_apply=$?"
timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "probe/" \
  -k regex:k_apply -c 2 -f -o /tmp/g23_smooth python tools/apply_probe.py --config 5 --reps 2 --op smooth > gpurun_out/g23_ncu_smooth.log 2>&1; echo "ncu_full=$?"
ncu -i /tmp/g23_smooth.ncu-rep --page raw --csv > gpurun_out/g23_smooth_raw.csv 2>/dev/null
ncu -i /tmp/g23_smooth.ncu-rep --page details --csv > gpurun_out/g23_smooth_details.csv 2>/dev/null
ls -la gpurun_out/g23*
