set -u
mkdir -p gpurun_out
for sw in 0 -1; do
  timeout 600 python tools/solve_profile.py --config 5 --maxit 30 --warm 1 --sweep $sw > gpurun_out/g17_c5_sw$sw.log 2>&1
  timeout 600 python tools/solve_profile.py --config 3 --sweep $sw > gpurun_out/g17_c3_sw$sw.log 2>&1
done
timeout 900 ncu --nvtx --nvtx-include "mg/solve/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/g17_c5_solve_launches.csv python tools/solve_profile.py --config 5 --eager --maxit 3 --warm 1 > gpurun_out/g17_c5_ncu.log 2>&1; echo "ncu5=$?"
for f in gpurun_out/g17_*.log; do echo $f; cat $f; done
