set -u
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -k "not fullsize" --timeout 900 > gpurun_out/g35_pytest.log 2>&1; echo "pytest=$?"
grep -E "FAILED|passed|failed|Error" gpurun_out/g35_pytest.log | tail -8
