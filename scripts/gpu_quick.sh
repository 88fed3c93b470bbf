# quick iteration: GPU tests + C2 and T benches (both algorithms)
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for cfg in C2 T; do
  st=10; [ $cfg = T ] && st=3
  timeout 900 python bench.py --config $cfg --steps $st --warmup 3 --no-oracle $EXTRA > gpurun_out/q_${cfg}.json 2>/dev/null
  python -c "
import json;d=json.load(open('gpurun_out/q_${cfg}.json'))
for a,r in d['per_algo'].items(): print('$cfg', a, 'ms %.2f'%r['ms'], 'Ge/s %.2f'%(r['edges_per_s']/1e9), {k:round(x,2) for k,x in r['kernel_ms_per_step'].items()}, 'frac %.3f'%r['roofline']['frac'])
print('   e2e ms %.1f'%d['e2e']['ms_per_step'])"
done
