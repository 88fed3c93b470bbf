cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_parity.py tests/test_capi.py -m gpu -x -q 2>&1 | tail -1
for cfg in C2 C3 T; do timeout 300 python scripts/po_profile.py $cfg 0 2>&1 | grep -v "level sizes"; done
for v in h8 h128; do
  for cfg in C2 T; do
    PICO_LIB=build_variants/libpico_$v.so timeout 300 python scripts/po_profile.py $cfg 0 2>&1 | grep "levels.*subrounds" | sed "s/^/$v /" | grep -o "^[a-z0-9]* [CT][0-9]* \|'peel': [0-9.]*" | tr '\n' ' '; echo
  done
done
