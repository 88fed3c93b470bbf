cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_parity.py -m gpu -x -q -k "peel or corpus or fixture or rmat" 2>&1 | tail -1
for v in b1 b8 b32 b128 b32u4; do
  for cfg in C2 T; do
    PICO_LIB=build_variants/libpico_$v.so timeout 300 python scripts/po_profile.py $cfg 0 2>&1 | grep "levels.*subrounds" | sed "s/^/$v /" | grep -o "^[a-z0-9]* [CT][0-9]* \|'peel': [0-9.]*" | tr '\n' ' '; echo
  done
done
timeout 300 python scripts/po_profile.py T 0 2>&1 | grep -v "level sizes"
