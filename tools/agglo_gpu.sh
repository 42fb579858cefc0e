mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_agglomerate.py -q > gpurun_out/r02_pytest_agglo.log 2>&1; echo "pytest=$?"; tail -3 gpurun_out/r02_pytest_agglo.log
timeout 900 python tools/agglo_probe.py > gpurun_out/r02_agglo_probe.jsonl 2>&1; echo "probe=$?"; cat gpurun_out/r02_agglo_probe.jsonl | cut -c1-300
