set -u
mkdir -p gpurun_out
L=paper_1811_09909_b200
cp $L/libmgdtn.so /tmp/early.so
for v in early late; do
  cp /tmp/$v.so $L/libmgdtn.so 2>/dev/null || cp $L/libmgdtn_late.so $L/libmgdtn.so
  for c in 2 4 3; do timeout 600 python tools/solve_profile.py --config $c > gpurun_out/g16_${v}_c$c.log 2>&1; done
  timeout 600 python tools/solve_profile.py --config 5 --maxit 30 --warm 1 > gpurun_out/g16_${v}_c5.log 2>&1
done
for f in gpurun_out/g16_*.log; do echo $f; cat $f; done
