set -u
mkdir -p gpurun_out
for v in 4 2; do
  MGDTN_ORBW=$v timeout 600 python tools/solve_profile.py --config 5 --maxit 30 --warm 1 > gpurun_out/g40_c5_w$v.log 2>&1
done
MGDTN_ORBW=4 timeout 900 ncu --nvtx --nvtx-include "mg/solve/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/g40_c5.csv python tools/solve_profile.py --config 5 --eager --maxit 3 --warm 1 > /dev/null 2>&1
python tools/iter_profile.py gpurun_out/g40_c5.csv > gpurun_out/g40_c5_iter.txt 2>&1
MGDTN_ORBW=4 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "c2 or c5" --timeout 600 > gpurun_out/g40_pytest.log 2>&1; echo "pytest=$?"
grep -E "FAILED|passed|failed|Error" gpurun_out/g40_pytest.log | tail -3
for f in gpurun_out/g40_c5_w*.log; do echo "$f $(tail -n 1 $f)"; done
grep "k_apply_orb2\|iteration" gpurun_out/g40_c5_iter.txt
