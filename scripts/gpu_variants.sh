# A/B: shadow width x L2 hints, HistoCore on C2 and T (default push/pull choice)
cd $GRAFT_REPO_ROOT
for cfg in C2 T; do
  for v in s16_h0 s16_h1 s8_h0 s8_h1; do
    st=10; [ $cfg = T ] && st=3
    PICO_LIB=build_variants/libpico_$v.so timeout 600 python bench.py --config $cfg --steps $st --warmup 3 --no-oracle --no-both > gpurun_out/var_${cfg}_$v.json 2>/dev/null
    python -c "
import json;d=json.load(open('gpurun_out/var_${cfg}_$v.json'));r=d['per_algo']['histocore']
print('$cfg $v', 'ms %.2f'%r['ms'], {k:round(x,2) for k,x in r['kernel_ms_per_step'].items()})"
  done
done
