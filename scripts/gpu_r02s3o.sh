# init warp-class split at d = 1024 (and 512): A/B of HistoCore per-kernel times, same box
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for cfg in T C4 C2 C3; do
  for v in base wsplit ws512; do
    PICO_LIB=build_variants/libpico_$v.so timeout 900 python bench.py --config $cfg --steps 3 --warmup 3 --no-oracle --extras '' --no-both > gpurun_out/s3o_${cfg}_$v.json 2> gpurun_out/s3o_${cfg}_$v.log
    echo "$cfg $v $(grep 'histocore:' gpurun_out/s3o_${cfg}_$v.log | grep -o "[0-9.]* ms/step\|'init': [0-9.]*")"
  done
done
