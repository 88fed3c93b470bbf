cd $GRAFT_REPO_ROOT
O=gpurun_out/r02h; mkdir -p $O
for v in s1 s2 s4 s8; do
  for cfg in C2 T; do
    PICO_LIB=build_variants/libpico_$v.so timeout 300 python scripts/po_profile.py $cfg 0 2>&1 | grep levels | sed "s/^/$v /"
  done
done
