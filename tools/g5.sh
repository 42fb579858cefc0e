set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/g5_pytest.log 2>&1; echo "pytest=$?"
tail -3 gpurun_out/g5_pytest.log
timeout 300 python tools/solve_profile.py --config 2 > gpurun_out/g5_c2.log 2>&1; echo "c2=$?"
timeout 600 python tools/solve_profile.py --config 5 --maxit 30 --warm 1 > gpurun_out/g5_c5.log 2>&1; echo "c5=$?"
timeout 900 ncu --nvtx --nvtx-include "mg/solve/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/g5_c5_solve_launches.csv python tools/solve_profile.py --config 5 --eager --maxit 3 --warm 1 > gpurun_out/g5_c5_ncu.log 2>&1; echo "ncu5=$?"
cat gpurun_out/g5_c2.log gpurun_out/g5_c5.log
