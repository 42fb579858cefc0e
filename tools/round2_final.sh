#!/bin/bash
# End-of-round-2 measurement (no profiler): GPU suite, smoke, default bench line (config 5).
set -u
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r02_pytest_gpu_head.log 2>&1; echo "pytest=$?"
tail -3 gpurun_out/r02_pytest_gpu_head.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke_head.log 2>&1; echo "smoke=$?"
tail -2 gpurun_out/r02_smoke_head.log
timeout 900 python bench.py > gpurun_out/r02_bench_head.log 2>&1; echo "bench=$?"
grep '^{' gpurun_out/r02_bench_head.log | cut -c1-600
