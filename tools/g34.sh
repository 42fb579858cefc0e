set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_partition.py -m gpu -q -x --timeout 600 > gpurun_out/g34_pytest.log 2>&1; echo "pytest=$?"
grep -E "FAILED|passed|failed|Error" gpurun_out/g34_pytest.log | tail -8
for c in 2 3 4; do
  for g in 0 16384 65536 262144 1048576; do
    timeout 600 python tools/solve_profile.py --config $c --opt 4=$g > gpurun_out/g34_c${c}_g$g.log 2>&1
  done
done
for g in 0 65536 4194304; do
  timeout 600 python tools/solve_profile.py --config 5 --maxit 30 --warm 1 --opt 4=$g > gpurun_out/g34_c5_g$g.log 2>&1
done
for f in gpurun_out/g34_c*.log; do echo "$f $(tail -n 1 $f)"; done
