set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "exec_path" --timeout 300 > gpurun_out/g28_pytest.log 2>&1; echo "pytest=$?"
grep -E "PASS|FAIL|passed|failed|Error" gpurun_out/g28_pytest.log | tail -15
for c in 5 3; do
  for sw in -1 1; do
    timeout 600 python tools/solve_profile.py --config $c --maxit 30 --warm 1 --sweep $sw > gpurun_out/g28_c${c}_sw$sw.log 2>&1; echo "c$c sw$sw=$?"
  done
done
tail -n 3 gpurun_out/g28_c*.log
