# A/B of env-selected kernel variants on the bench step: tools/ab_env.sh "<env1>" "<env2>" ...
for cfg in ${CFGS:-2 4}; do
  for e in "$@"; do
    env $e timeout 300 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | grep '^{' | \
      python -c "import sys,json; d=json.loads(sys.stdin.read()); print('c$cfg', '$e', 'value %.4g'%d['value'], 'iters', d['iters'], 'solve %.3f'%d['phases_ms']['solve'], 'setup %.3f'%d['phases_ms']['setup'], 'apply %.2f us'%(1e3*d['phases_ms']['fine_apply']))"
  done
done
