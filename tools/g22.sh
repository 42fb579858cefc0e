set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/g22_pytest.log 2>&1; echo "pytest=$?"
grep -E "FAILED|passed|failed" gpurun_out/g22_pytest.log | tail -8
timeout 600 python tools/solve_profile.py --config 5 --maxit 30 --warm 1 > gpurun_out/g22_c5.log 2>&1; cat gpurun_out/g22_c5.log
