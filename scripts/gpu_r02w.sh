cd $GRAFT_REPO_ROOT
for fl in 0 512; do
  timeout 600 python scripts/round_profile.py --config T --reps 1 --flags $fl 2>&1 | head -1 | cut -c1-250
  timeout 300 python scripts/po_profile.py T $fl 2>&1 | grep "levels.*subrounds" | grep -o "'peel'.*\|kmax [0-9]*"
  timeout 300 python scripts/po_profile.py C4 $fl 2>&1 | grep "levels.*subrounds" | grep -o "'peel'.*\|kmax [0-9]*"
done
