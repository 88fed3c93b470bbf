cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for cfg in C2 T; do
  for v in seg32 seg64 seg256; do
    for fl in 0 64; do
    st=10; [ $cfg = T ] && st=3
    PICO_LIB=build_variants/libpico_$v.so timeout 600 python bench.py --config $cfg --steps $st --warmup 3 --no-oracle --no-both --flags $fl > gpurun_out/var_${cfg}_${v}_$fl.json 2>/dev/null
    python -c "
import json;d=json.load(open('gpurun_out/var_${cfg}_${v}_$fl.json'));r=d['per_algo']['histocore']
print('$cfg $v flags $fl', 'ms %.2f'%r['ms'], {k:round(x,2) for k,x in r['kernel_ms_per_step'].items()})"
    done
  done
done
