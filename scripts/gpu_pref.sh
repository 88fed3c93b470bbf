cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for cfg in C2 T; do
  for fl in 0 2048; do
    st=10; [ $cfg = T ] && st=3
    timeout 600 python bench.py --config $cfg --steps $st --warmup 3 --no-oracle --no-both --flags $fl > gpurun_out/pref_${cfg}_$fl.json 2>/dev/null
    python -c "
import json;d=json.load(open('gpurun_out/pref_${cfg}_$fl.json'));r=d['per_algo']['histocore']
print('$cfg flags $fl', 'ms %.2f'%r['ms'], {k:round(x,2) for k,x in r['kernel_ms_per_step'].items()}, 'arcs', r['stats']['arcs_scanned'], 'guard', r['stats']['guarded_arcs'], 'frac %.3f'%r['roofline']['frac'])"
  done
done
