set -u
mkdir -p gpurun_out
timeout 600 python tools/apply_probe.py --config 5 --reps 3 > gpurun_out/g7_plain.log 2>&1; echo "plain=$?"
timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "probe/" \
  -k regex:k_apply_sweep -c 1 -f -o /tmp/g7_sweep python tools/apply_probe.py --config 5 --reps 3 > gpurun_out/g7_ncu.log 2>&1; echo "ncu=$?"
ncu -i /tmp/g7_sweep.ncu-rep --page raw --csv > gpurun_out/g7_sweep_raw.csv 2>/dev/null
ncu -i /tmp/g7_sweep.ncu-rep --page details --csv > gpurun_out/g7_sweep_details.csv 2>/dev/null
ncu -i /tmp/g7_sweep.ncu-rep --page source --csv --print-source sass > gpurun_out/g7_sweep_source.csv 2>/dev/null
ls -la gpurun_out/g7*
