cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
summ() { python - "$1" <<'PY'
import json,sys
d=json.load(open(sys.argv[1]))
for a,r in d['per_algo'].items():
    print(sys.argv[1].split('/')[-1], a, 'ms %.2f'%r['ms'], 'Ge/s %.3f'%(r['edges_per_s']/1e9), 'l2',r['rounds_l2'],'lv',r['levels'], 'frac %.3f'%r['roofline']['frac'], 'pull',r['stats'].get('pull_rounds'), {k:round(v,2) for k,v in r['kernel_ms_per_step'].items()})
print('   parity', d['parity'], 'e2e ms %.1f'%d['e2e']['ms_per_step'])
PY
}
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.log; summ gpurun_out/bench_c2.json
timeout 600 python bench.py --steps 10 --warmup 3 --no-oracle --no-both --flags 64 > gpurun_out/bench_c2_push.json 2>/dev/null; summ gpurun_out/bench_c2_push.json
timeout 900 python bench.py --config T --steps 3 --warmup 3 --no-oracle > gpurun_out/bench_T.json 2> gpurun_out/bench_T.log; summ gpurun_out/bench_T.json
