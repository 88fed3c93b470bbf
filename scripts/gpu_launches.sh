# per-kernel launch list (ncu gpu__time_duration, cold-cache, serialised) of one call
cd $GRAFT_REPO_ROOT
CFG=${CFG:-T}
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"${KRE:-hc_|po_|rl_|Device}" -c ${NC:-40} --csv --log-file gpurun_out/launches_${CFG}.csv python scripts/round_profile.py --config $CFG --reps 1 ${RPFLAGS} > /dev/null 2>&1
echo ncu=$?
