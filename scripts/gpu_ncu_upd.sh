# ncu --set full of the first host-loop UpdateHisto launch (round 1) for library variants
cd $GRAFT_REPO_ROOT
CFG=${CFG:-T}
for v in ${VARIANTS:-main}; do
  lib=""; [ "$v" != main ] && lib=build_variants/libpico_$v.so
  PICO_LIB=$lib timeout 900 ncu --set full --clock-control none --import-source on -k regex:"hc_update" -c ${NC:-1} \
    -o gpurun_out/prof_${CFG}_upd_$v python scripts/round_profile.py --config $CFG --flags $((8 + ${XFLAGS:-0})) --reps 1 > gpurun_out/ncu_${CFG}_upd_$v.log 2>&1
  echo ncu $v=$?
done
