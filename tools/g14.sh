set -u
mkdir -p gpurun_out
for v in graph eager; do
  if [ $v = eager ]; then E=--eager; else E=; fi
  timeout 600 python tools/solve_profile.py --config 5 --maxit 30 --warm 1 $E > gpurun_out/g14_$v.log 2>&1; echo "$v=$?"
done
MGDTN_PDL=0 timeout 600 python tools/solve_profile.py --config 5 --maxit 30 --warm 1 > gpurun_out/g14_nopdl.log 2>&1; echo "nopdl=$?"
nvidia-smi --query-gpu=power.limit,power.draw,clocks.sm,clocks.mem --format=csv > gpurun_out/g14_smi.txt
cat gpurun_out/g14_*.log gpurun_out/g14_smi.txt
