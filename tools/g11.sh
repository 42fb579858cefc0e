set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/g11_pytest.log 2>&1; echo "pytest=$?"
grep -E "FAILED|passed|failed" gpurun_out/g11_pytest.log | tail -40
