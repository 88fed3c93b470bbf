# per-round profiles (scripts/round_profile.py) of C2 and T
cd $GRAFT_REPO_ROOT
for cfg in ${CFGS:-C2 T}; do
  timeout 600 python scripts/round_profile.py --config $cfg ${RPFLAGS} 2>&1 | tee gpurun_out/rp_${cfg}.txt
done
