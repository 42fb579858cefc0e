set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_c5_recipe.py tests/test_gpu_paper_tables.py tests/test_gpu_partition.py -m gpu -q -x --timeout 600 > gpurun_out/g36_pytest.log 2>&1; echo "pytest=$?"
grep -E "FAILED|passed|failed|Error" gpurun_out/g36_pytest.log | tail -5
timeout 600 python tools/solve_profile.py --config 5 --maxit 30 --warm 1 > gpurun_out/g36_c5.log 2>&1
for c in 2 3 4; do timeout 600 python tools/solve_profile.py --config $c > gpurun_out/g36_c$c.log 2>&1; done
timeout 900 ncu --nvtx --nvtx-include "mg/solve/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/g36_c5_solve_launches.csv python tools/solve_profile.py --config 5 --eager --maxit 3 --warm 1 > gpurun_out/g36_c5_ncu.log 2>&1; echo "ncu5=$?"
python tools/iter_profile.py gpurun_out/g36_c5_solve_launches.csv > gpurun_out/g36_c5_iter.txt 2>&1
tail -3 gpurun_out/g36_c5_iter.txt
for f in gpurun_out/g36_c*.log; do echo "$f $(tail -n 1 $f)"; done
