set -u
mkdir -p gpurun_out
L=paper_1811_09909_b200
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 600 > gpurun_out/g38_pytest.log 2>&1; echo "pytest=$?"
grep -E "FAILED|passed|failed|Error" gpurun_out/g38_pytest.log | tail -5
for v in 0 1; do MGDTN_ORB2=$v timeout 600 python tools/solve_profile.py --config 5 --maxit 30 --warm 1 > gpurun_out/g38_c5_orb2_$v.log 2>&1; done
MGDTN_ORB2=1 timeout 900 ncu --nvtx --nvtx-include "mg/solve/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/g38_c5_A.csv python tools/solve_profile.py --config 5 --eager --maxit 3 --warm 1 > /dev/null 2>&1
python tools/iter_profile.py gpurun_out/g38_c5_A.csv > gpurun_out/g38_c5_A_iter.txt 2>&1
cp $L/libmgdtn_b.so.tmp $L/libmgdtn.so
MGDTN_ORB2=1 timeout 600 python tools/solve_profile.py --config 5 --maxit 30 --warm 1 > gpurun_out/g38_c5_orb2_B.log 2>&1
MGDTN_ORB2=1 timeout 900 ncu --nvtx --nvtx-include "mg/solve/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/g38_c5_B.csv python tools/solve_profile.py --config 5 --eager --maxit 3 --warm 1 > /dev/null 2>&1
python tools/iter_profile.py gpurun_out/g38_c5_B.csv > gpurun_out/g38_c5_B_iter.txt 2>&1
for f in gpurun_out/g38_c5_orb2*.log; do echo "$f $(tail -n 1 $f)"; done
grep "k_apply_orb2\|iteration" gpurun_out/g38_c5_A_iter.txt gpurun_out/g38_c5_B_iter.txt
