# profile T in host-loop mode: per-launch times, then full sets of round-1/2 updates (push vs pull)
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 600 python bench.py --steps 10 --warmup 3 --no-oracle > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.log; grep "\[bench\]" gpurun_out/bench_c2.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:"hc_" --csv --log-file gpurun_out/launches_T_hostloop.csv python bench.py --config T --steps 1 --warmup 3 --no-oracle --no-both --flags 8 > /dev/null 2>&1; echo ncuT=$?
timeout 900 ncu --set full --clock-control none -k regex:"hc_update" -s 0 -c 3 -o gpurun_out/prof_T_push python bench.py --config T --steps 1 --warmup 3 --no-oracle --no-both --flags 72 > /dev/null 2>&1; echo ncuPush=$?
timeout 900 ncu --set full --clock-control none -k regex:"hc_update" -s 0 -c 3 -o gpurun_out/prof_T_pull python bench.py --config T --steps 1 --warmup 3 --no-oracle --no-both --flags 136 > /dev/null 2>&1; echo ncuPull=$?
timeout 900 ncu --set full --clock-control none -k regex:"hc_init|hc_degree|hc_shadow" -c 6 -o gpurun_out/prof_T_init python bench.py --config T --steps 1 --warmup 3 --no-oracle --no-both > /dev/null 2>&1; echo ncuInit=$?
