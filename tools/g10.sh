set -u
mkdir -p gpurun_out
timeout 600 python bench.py --config 2 --steps 5 --warmup 3 > gpurun_out/g10_b2.log 2>&1; echo "b2=$?"
timeout 1200 python bench.py --steps 2 --warmup 1 > gpurun_out/g10_b5.log 2>&1; echo "b5=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/g10_ref.log 2>&1; echo "ref=$?"
tail -c 3000 gpurun_out/g10_b2.log; tail -c 3000 gpurun_out/g10_b5.log; tail -c 1500 gpurun_out/g10_ref.log
