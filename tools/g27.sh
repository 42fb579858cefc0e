set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_invariants.py tests/test_gpu_c5_recipe.py -m gpu -q -v --timeout 300 > gpurun_out/g27_pytest.log 2>&1; echo "pytest=$?"
grep -E "PASS|FAIL|passed|failed|Error" gpurun_out/g27_pytest.log | tail -15
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_peak tools/fp64_peak.cu && /tmp/fp64_peak > gpurun_out/g27_fp64.json; cat gpurun_out/g27_fp64.json
timeout 600 python bench.py --config 2 --steps 10 --warmup 3 > gpurun_out/g27_b2.log 2>&1; echo b2=$?
timeout 900 python bench.py --config 3 --steps 3 --warmup 3 > gpurun_out/g27_b3.log 2>&1; echo b3=$?
timeout 600 python bench.py --config 4 --steps 5 --warmup 3 > gpurun_out/g27_b4.log 2>&1; echo b4=$?
timeout 600 python bench.py --config 1 --steps 10 --warmup 3 > gpurun_out/g27_b1.log 2>&1; echo b1=$?
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/g27_bench_launches.csv \
   python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/g27_bench_ncu.log 2>&1; echo ncu=$?
python tools/agg_launches.py gpurun_out/g27_bench_launches.csv 60 > gpurun_out/g27_bench_launches_summary.txt
