set -u
mkdir -p gpurun_out
timeout 600 python tools/apply_probe.py --config 5 --op smooth --steps 2 --reps 3 > gpurun_out/g37_probe.log 2>&1; echo probe=$?
cat gpurun_out/g37_probe.log | tail -2
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_apply_orb --launch-skip 6 -c 2 \
  -o gpurun_out/g37_smooth python tools/apply_probe.py --config 5 --op smooth --steps 2 --reps 1 > gpurun_out/g37_ncu.log 2>&1; echo ncu=$?
tail -5 gpurun_out/g37_ncu.log
