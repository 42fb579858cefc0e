set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_partition.py tests/test_gpu_transfer*.py -m gpu -q -x > gpurun_out/g31_pytest.log 2>&1; echo "pytest=$?"
grep -E "FAILED|passed|failed" gpurun_out/g31_pytest.log | tail -5
for c in 2 3; do timeout 600 python tools/solve_profile.py --config $c --maxit 30 --warm 1 > gpurun_out/g31_c$c.log 2>&1; done
timeout 600 python tools/solve_profile.py --config 5 --maxit 30 --warm 1 > gpurun_out/g31_c5.log 2>&1
timeout 900 ncu --nvtx --nvtx-include "mg/solve/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/g31_c5_solve_launches.csv python tools/solve_profile.py --config 5 --eager --maxit 3 --warm 1 > gpurun_out/g31_c5_ncu.log 2>&1; echo "ncu5=$?"
python tools/iter_profile.py gpurun_out/g31_c5_solve_launches.csv > gpurun_out/g31_c5_iter.txt 2>&1
grep -E "prolong|iteration" gpurun_out/g31_c5_iter.txt
cat gpurun_out/g31_c*.log
