cd $GRAFT_REPO_ROOT
for v in base p16 p64; do
  if [ $v = base ]; then L=""; else L="PICO_LIB=build_variants/libpico_$v.so"; fi
  env $L timeout 600 python scripts/round_profile.py --config T --reps 1 2>&1 | head -1 | cut -c20-250 | sed "s/^/$v /"
  env $L timeout 600 python scripts/round_profile.py --config T --reps 1 2>&1 | sed -n 3,12p | awk '{print $1, $5}' | tr '\n' ' '; echo
done
