set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_partition.py tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/g13_pytest.log 2>&1; echo "pytest=$?"
grep -E "FAILED|passed|failed|Error" gpurun_out/g13_pytest.log | tail -20
