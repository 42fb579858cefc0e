set -u
mkdir -p gpurun_out
for pf in 0 17 2 18 34 33 1; do
  timeout 600 python tools/solve_profile.py --config 5 --maxit 30 --warm 1 --opt 4=$pf > gpurun_out/g30_c5_pf$pf.log 2>&1; echo "c5 pf$pf=$?"
done
for f in gpurun_out/g30_c5_*.log; do echo $f; tail -n 1 $f; done
