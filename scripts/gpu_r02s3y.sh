# edge-list fill occupancy A/B (launch-bounds min CTAs 1 / 6 / 8), same box
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/s3y
for rep in 1 2; do
for cfg in T C4; do
  for v in fill1 fill6 fill8; do
    PICO_LIB=build_variants/libpico_$v.so timeout 900 python bench.py --config $cfg --steps 3 --warmup 3 --no-oracle --extras '' --no-both > gpurun_out/s3y/${cfg}_$v.json 2> gpurun_out/s3y/${cfg}_$v.log
    echo "$cfg $v $(grep 'histocore:' gpurun_out/s3y/${cfg}_$v.log | grep -o "[0-9.]* ms/step\|'edgelist': [0-9.]*")"
  done
done
done
