set -x
for g in bal full dyn; do
  for c in 2 3 4; do
    MGDTN_GRID=$g timeout 120 python tools/apply_probe.py --config $c --reps 30 2>&1 | tail -1 | sed "s/^/$g c$c /"
  done
done
MGDTN_GRID=dyn timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "c2n64 or c4n64 or c3n64" 2>&1 | tail -2
for g in bal full dyn; do
  MGDTN_GRID=$g timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$g', 'value %.4g'%d['value'], 'solve %.3f'%d['phases_ms']['solve'], 'apply %.2f us'%(1e3*d['phases_ms']['fine_apply']), 'frac %.3f'%d['roofline']['frac'])"
done
