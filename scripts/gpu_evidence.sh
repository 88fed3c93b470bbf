# full evidence run: tests, default bench (with oracle), launch list, ncu --set full of the step kernels
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.log; echo bench=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"hc_|po_|rl_|max_kernel" --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-oracle > /dev/null 2>&1; echo ncu1=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"hc_|po_" -c 12 -o gpurun_out/prof_c2_full python bench.py --steps 1 --warmup 0 --no-oracle > gpurun_out/ncu_full.log 2>&1; echo ncu2=$?
timeout 900 python bench.py --config T --steps 3 --warmup 3 --no-oracle > gpurun_out/bench_T.json 2> gpurun_out/bench_T.log; echo benchT=$?
timeout 900 ncu --set full --clock-control none -k regex:"hc_rounds|po_levels|hc_init|rl_" -c 10 -o gpurun_out/prof_T_full python bench.py --config T --steps 1 --warmup 0 --no-oracle > gpurun_out/ncu_T.log 2>&1; echo ncu3=$?
