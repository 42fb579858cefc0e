set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_c5_recipe.py -m gpu -q -x --timeout 600 > gpurun_out/g39_pytest.log 2>&1; echo "pytest=$?"
grep -E "FAILED|passed|failed|Error" gpurun_out/g39_pytest.log | tail -5
for v in 1 0; do
  MGDTN_ORB2=$v timeout 600 python tools/solve_profile.py --config 5 --maxit 30 --warm 1 > gpurun_out/g39_c5_orb2_$v.log 2>&1
  MGDTN_ORB2=$v timeout 600 python tools/solve_profile.py --config 4 > gpurun_out/g39_c4_orb2_$v.log 2>&1
  MGDTN_ORB2=$v timeout 600 python tools/solve_profile.py --config 2 > gpurun_out/g39_c2_orb2_$v.log 2>&1
done
timeout 900 ncu --nvtx --nvtx-include "mg/solve/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/g39_c5.csv python tools/solve_profile.py --config 5 --eager --maxit 3 --warm 1 > /dev/null 2>&1
python tools/iter_profile.py gpurun_out/g39_c5.csv > gpurun_out/g39_c5_iter.txt 2>&1
for f in gpurun_out/g39_c*orb2*.log; do echo "$f $(tail -n 1 $f)"; done
grep "k_apply_orb\|iteration" gpurun_out/g39_c5_iter.txt | head -12; tail -1 gpurun_out/g39_c5_iter.txt
