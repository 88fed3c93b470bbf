cd $GRAFT_REPO_ROOT
for v in loop16 loop32; do for cfg in T C4 C2; do
  PICO_LIB=build_variants/libpico_$v.so timeout 300 python scripts/peel_stress.py $cfg 80 2>&1 | tail -1
done; done
