set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_c5_recipe.py tests/test_gpu_paper_tables.py -m gpu -q -x --timeout 600 > gpurun_out/g33_pytest.log 2>&1; echo "pytest=$?"
grep -E "FAILED|passed|failed" gpurun_out/g33_pytest.log | tail -5
timeout 600 python tools/solve_profile.py --config 5 --maxit 30 --warm 1 > gpurun_out/g33_c5.log 2>&1
for c in 2 3 4; do timeout 600 python tools/solve_profile.py --config $c > gpurun_out/g33_c$c.log 2>&1; done
for c in 2 3; do
 for ne in 1024 4096 16384; do
  for cl in 8 16; do
   MGDTN_TAIL_NE=$ne MGDTN_TAIL_CLUSTER=$cl timeout 300 python tools/solve_profile.py --config $c > gpurun_out/g33_tail_c${c}_ne${ne}_cl${cl}.log 2>&1
  done
 done
done
for f in gpurun_out/g33_c*.log gpurun_out/g33_tail*.log; do echo "$f $(tail -n 1 $f)"; done
