# ncu evidence of the current code at T and C2: launch lists, --set full of the
# round kernel and the PeelOne level kernel (raw + source pages exported on the box)
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02e; mkdir -p $O
for cfg in C2 T; do
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"hc_|po_|rl_|max_kernel|DeviceScan" --csv --log-file $O/launches_${cfg}.csv python scripts/one_call.py $cfg > /dev/null 2>&1; echo launch_$cfg=$?
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"hc_rounds|hc_init|hc_el|po_levels|rl_arcs" -c 16 -o /tmp/prof_${cfg} python scripts/one_call.py $cfg > $O/ncu_$cfg.log 2>&1; echo ncu_$cfg=$?
  ncu -i /tmp/prof_${cfg}.ncu-rep --page raw --csv > $O/ncu_${cfg}_raw.csv 2>/dev/null
  ncu -i /tmp/prof_${cfg}.ncu-rep --page source --csv --kernel-name regex:hc_rounds --launch-count 1 > $O/ncu_${cfg}_rounds_source.csv 2>/dev/null
  ncu -i /tmp/prof_${cfg}.ncu-rep --page source --csv --kernel-name regex:po_levels --launch-count 1 > $O/ncu_${cfg}_peel_source.csv 2>/dev/null
done
cp /tmp/prof_C2.ncu-rep $O/ 2>/dev/null
du -sh $O
