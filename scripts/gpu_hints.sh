cd $GRAFT_REPO_ROOT
for cfg in C2 T; do
  for v in h0 h1; do
    st=10; [ $cfg = T ] && st=3
    PICO_LIB=build_variants/libpico_$v.so timeout 600 python bench.py --config $cfg --steps $st --warmup 3 --no-oracle --no-both > gpurun_out/var_${cfg}_${v}.json 2>/dev/null
    python -c "
import json;d=json.load(open('gpurun_out/var_${cfg}_${v}.json'));r=d['per_algo']['histocore']
print('$cfg $v', 'ms %.2f'%r['ms'], {k:round(x,2) for k,x in r['kernel_ms_per_step'].items()}, 'pull', r['stats']['pull_rounds'])"
  done
done
timeout 900 ncu --set full --clock-control none -k regex:"hc_update" -s 0 -c 2 -o gpurun_out/prof_T_upd python bench.py --config T --steps 1 --warmup 3 --no-oracle --no-both --flags 8 > /dev/null 2>&1; echo ncu=$?
