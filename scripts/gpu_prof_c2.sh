cd $GRAFT_REPO_ROOT
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:"hc_" --csv --log-file gpurun_out/launches_c2_hostloop.csv python bench.py --steps 1 --warmup 3 --no-oracle --no-both --flags 8 > /dev/null 2>&1; echo ncu1=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"hc_update|hc_collect" -s 0 -c 4 -o gpurun_out/prof_c2_upd python bench.py --steps 1 --warmup 0 --no-oracle --no-both --flags 8 > /dev/null 2>&1; echo ncu2=$?
