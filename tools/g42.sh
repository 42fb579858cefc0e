set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_c5_recipe.py tests/test_gpu_partition.py -m gpu -q -x --timeout 600 > gpurun_out/g42_pytest.log 2>&1; echo "pytest=$?"
grep -E "FAILED|passed|failed|Error" gpurun_out/g42_pytest.log | tail -5
timeout 600 python tools/solve_profile.py --config 5 --maxit 30 --warm 1 > gpurun_out/g42_c5.log 2>&1
for c in 2 3 4; do timeout 600 python tools/solve_profile.py --config $c > gpurun_out/g42_c$c.log 2>&1; done
timeout 900 ncu --nvtx --nvtx-include "mg/solve/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/g42_c5.csv python tools/solve_profile.py --config 5 --eager --maxit 3 --warm 1 > /dev/null 2>&1
python tools/iter_profile.py gpurun_out/g42_c5.csv > gpurun_out/g42_c5_iter.txt 2>&1
for f in gpurun_out/g42_c*.log; do echo "$f $(tail -n 1 $f)"; done
grep "k_apply_orb<4\|k_apply_orb2\|iteration\|prolong" gpurun_out/g42_c5_iter.txt
