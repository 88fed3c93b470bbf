cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_parity.py -m gpu -x -q -k peel 2>&1 | tail -1
for rep in 1 2; do
for v in base head; do
  if [ $v = base ]; then L=""; else L="PICO_LIB=build_variants/libpico_$v.so"; fi
  for cfg in C1 C2 T; do env $L timeout 300 python scripts/po_profile.py $cfg 0 2>&1 | grep "levels.*subrounds" | grep -o "^[CT][0-9]* \|'peel': [0-9.]*" | tr '\n' ' '; echo $v; done
done
done
