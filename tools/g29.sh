set -u
mkdir -p gpurun_out
for c in 5 3 2; do
  for pf in 1 0; do
    timeout 600 python tools/solve_profile.py --config $c --maxit 30 --warm 1 --opt 4=$pf > gpurun_out/g29_c${c}_pf$pf.log 2>&1; echo "c$c pf$pf=$?"
  done
done
tail -n 2 gpurun_out/g29_c*.log
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 600 > gpurun_out/g29_pytest.log 2>&1; echo "pytest=$?"
grep -E "FAIL|passed|failed|Error" gpurun_out/g29_pytest.log | tail -15
