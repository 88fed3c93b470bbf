# ncu --set full of the first few host-loop UpdateHisto/SumHisto launches on T
cd $GRAFT_REPO_ROOT
CFG=${CFG:-T}
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"hc_update|hc_collect" -c ${NC:-4} \
  -o gpurun_out/prof_${CFG}_upd python scripts/round_profile.py --config $CFG --flags 8 --reps 1 > gpurun_out/ncu_${CFG}_upd.log 2>&1
echo ncu=$?
tail -3 gpurun_out/ncu_${CFG}_upd.log
