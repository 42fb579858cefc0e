set -u
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "probe/" \
  -k regex:k_apply_sweep -c 1 -f -o /tmp/g25 python tools/apply_probe.py --config 5 --level 12 --reps 2 --op smooth --sweep 1 --steps 2 > gpurun_out/g25_ncu.log 2>&1; echo "ncu=$?"
ncu -i /tmp/g25.ncu-rep --page details --csv > gpurun_out/g25_details.csv 2>/dev/null
ncu -i /tmp/g25.ncu-rep --page source --csv --print-source sass > gpurun_out/g25_source.csv 2>/dev/null
ls -la gpurun_out/g25*
