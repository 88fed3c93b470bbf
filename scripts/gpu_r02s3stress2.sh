# final-code stress: 200 PeelOne calls per config (the bench's timed-step call), results checked every 10
cd $GRAFT_REPO_ROOT
for cfg in T C4 C3 C2 C1; do timeout 600 python scripts/peel_stress.py $cfg 200 2>&1 | tail -1; done
