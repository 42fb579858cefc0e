#!/bin/bash
# End-of-round measurement, part 1 (no profiler): GPU suite, smoke, default bench line.
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r01_pytest_gpu_final.log 2>&1; echo "pytest=$?"
tail -3 gpurun_out/r01_pytest_gpu_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r01_smoke_final.log 2>&1; echo "smoke=$?"
tail -2 gpurun_out/r01_smoke_final.log
timeout 900 python bench.py > gpurun_out/r01_bench_final.log 2>&1; echo "bench=$?"
grep '^{' gpurun_out/r01_bench_final.log | cut -c1-400
