set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "exec_paths" --timeout 300 > gpurun_out/g24_pytest.log 2>&1; echo "pytest=$?"
tail -3 gpurun_out/g24_pytest.log
for sw in 1 -1; do
  timeout 600 python tools/solve_profile.py --config 5 --maxit 30 --warm 1 --sweep $sw > gpurun_out/g24_c5_sw$sw.log 2>&1
  timeout 600 python tools/solve_profile.py --config 3 --sweep $sw > gpurun_out/g24_c3_sw$sw.log 2>&1
done
cat gpurun_out/g24_c*.log
timeout 900 ncu --nvtx --nvtx-include "mg/solve/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/g24_c5_solve_launches.csv python tools/solve_profile.py --config 5 --eager --maxit 3 --warm 1 --sweep 1 > gpurun_out/g24_c5_ncu.log 2>&1; echo "ncu5=$?"
