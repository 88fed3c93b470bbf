cd $GRAFT_REPO_ROOT
for v in a2p3 a2p2 a4p2 u4p2 a8p2; do
  for cfg in C2 T; do
    PICO_LIB=build_variants/libpico_$v.so timeout 300 python scripts/po_profile.py $cfg 0 2>&1 | grep "levels.*subrounds" | sed "s/^/$v /" | grep -o "^[a-z0-9]* [CT][0-9]* \|'peel': [0-9.]*" | tr '\n' ' '; echo
  done
done
