set -u
mkdir -p gpurun_out
for c in 2 4 3; do
  timeout 600 python tools/solve_profile.py --config $c > gpurun_out/g15_c${c}_pdl.log 2>&1
  MGDTN_PDL=0 timeout 600 python tools/solve_profile.py --config $c > gpurun_out/g15_c${c}_nopdl.log 2>&1
done
cat gpurun_out/g15_*.log
