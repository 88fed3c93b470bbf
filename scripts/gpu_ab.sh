# GPU tests + per-round profiles of library variants: VARIANTS="main noagg ..." CFGS="C2 T"
cd $GRAFT_REPO_ROOT
if [ -z "$NOTEST" ]; then timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3; fi
for cfg in ${CFGS:-C2 T}; do
  for v in ${VARIANTS:-main}; do
    lib=""; [ "$v" != main ] && lib=build_variants/libpico_$v.so
    echo "=== $cfg $v"
    PICO_LIB=$lib timeout 600 python scripts/round_profile.py --config $cfg $RPFLAGS 2>&1 > gpurun_out/rp_${cfg}_$v.txt
    head -1 gpurun_out/rp_${cfg}_$v.txt; tail -1 gpurun_out/rp_${cfg}_$v.txt
  done
done
