set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/g1_smi.txt
timeout 600 python tools/solve_profile.py --config 5 --eager --maxit 5 --warm 1 > gpurun_out/g1_c5_plain.log 2>&1; echo "plain5=$?"
timeout 900 ncu --nvtx --nvtx-include "mg/solve/" --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/g1_c5_solve_launches.csv python tools/solve_profile.py --config 5 --eager --maxit 5 --warm 1 > gpurun_out/g1_c5_ncu.log 2>&1; echo "ncu5=$?"
python tools/agg_launches.py gpurun_out/g1_c5_solve_launches.csv 80 > gpurun_out/g1_c5_solve_summary.txt
timeout 300 python tools/solve_profile.py --config 2 --eager > gpurun_out/g1_c2_plain.log 2>&1; echo "plain2=$?"
timeout 300 python tools/solve_profile.py --config 2 > gpurun_out/g1_c2_graph.log 2>&1; echo "graph2=$?"
timeout 600 ncu --nvtx --nvtx-include "mg/solve/" --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/g1_c2_solve_launches.csv python tools/solve_profile.py --config 2 --eager > gpurun_out/g1_c2_ncu.log 2>&1; echo "ncu2=$?"
python tools/agg_launches.py gpurun_out/g1_c2_solve_launches.csv 80 > gpurun_out/g1_c2_solve_summary.txt
