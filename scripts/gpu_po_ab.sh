# PeelOne A/B over library variants: VARIANTS="main ..." CFGS="C2 T"
cd $GRAFT_REPO_ROOT
for cfg in ${CFGS:-C2 T}; do
  for v in ${VARIANTS:-main}; do
    lib=""; [ "$v" != main ] && lib=build_variants/libpico_$v.so
    echo "=== $cfg $v"
    PICO_LIB=$lib timeout 300 python scripts/po_profile.py $cfg 2>&1 | head -1
  done
done
