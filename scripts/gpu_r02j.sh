cd $GRAFT_REPO_ROOT
for cfg in C2 T; do timeout 300 python scripts/po_profile.py $cfg 0 2>&1 | grep -v "^level sizes" | grep slowest; done
