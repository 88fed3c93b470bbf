set -x
cd $GRAFT_REPO_ROOT
lscpu | grep -E "Model name|^CPU\(s\)" > gpurun_out/host.txt
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.log; echo rc=$?
tail -3 gpurun_out/bench_c2.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"hc_|po_|max_kernel" --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-oracle > /dev/null 2>&1; echo ncu1=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"hc_rounds|hc_init|po_levels" -c 6 -o gpurun_out/prof_c2 python bench.py --steps 1 --warmup 3 --no-oracle > gpurun_out/ncu_full.log 2>&1; echo ncu2=$?
tail -5 gpurun_out/ncu_full.log
timeout 900 python bench.py --config T --steps 3 --warmup 3 --no-oracle > gpurun_out/bench_T.json 2> gpurun_out/bench_T.log; echo rcT=$?
tail -3 gpurun_out/bench_T.log
