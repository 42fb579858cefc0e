set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_partition.py -m gpu -q -x --timeout 300 > gpurun_out/g21_pytest.log 2>&1; echo "pytest=$?"
tail -5 gpurun_out/g21_pytest.log
