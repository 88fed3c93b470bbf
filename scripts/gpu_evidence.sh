# full evidence run: tests, benches of every single-GPU config, launch lists,
# ncu --set full of the step kernels (C2, T), exported to CSV on the box
# (gpurun brings back at most 64 MiB)
cd $GRAFT_REPO_ROOT
R=${R:-r01}
O=gpurun_out/$R
mkdir -p $O
lscpu | grep -E "Model name|^CPU\(s\)" > $O/host.txt
if [ -z "$NOTEST" ]; then timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2; fi
if [ -z "$NOBENCH" ]; then
timeout 900 python bench.py > $O/bench_C2.json 2> $O/bench_C2.log; echo bench_C2=$?
for cfg in C1 C3; do
  timeout 900 python bench.py --config $cfg --steps 10 > $O/bench_$cfg.json 2> $O/bench_$cfg.log; echo bench_$cfg=$?
done
for cfg in ${BIG:-T C4}; do
  timeout 1200 python bench.py --config $cfg --steps 3 --no-oracle > $O/bench_$cfg.json 2> $O/bench_$cfg.log; echo bench_$cfg=$?
  tail -3 $O/bench_$cfg.log
done
fi
if [ -z "$NONCU" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"hc_|po_|rl_|max_kernel" --csv --log-file $O/launches_C2.csv python scripts/one_call.py C2 > /dev/null 2>&1; echo ncu_launch_C2=$?
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"hc_|po_|rl_|max_kernel" --csv --log-file $O/launches_T.csv python scripts/one_call.py T > /dev/null 2>&1; echo ncu_launch_T=$?
for cfg in C2 T; do
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"hc_rounds|hc_init|hc_el|po_levels|rl_arcs" -c 16 -o /tmp/prof_${cfg} python scripts/one_call.py $cfg > $O/ncu_$cfg.log 2>&1; echo ncu_$cfg=$?
  ncu -i /tmp/prof_${cfg}.ncu-rep --page raw --csv > $O/ncu_${cfg}_raw.csv 2>/dev/null
  ncu -i /tmp/prof_${cfg}.ncu-rep --page details --csv > $O/ncu_${cfg}_details.csv 2>/dev/null
  ncu -i /tmp/prof_${cfg}.ncu-rep --page source --csv --kernel-name regex:hc_rounds --launch-count 1 > $O/ncu_${cfg}_rounds_source.csv 2>/dev/null
  ls -la /tmp/prof_${cfg}.ncu-rep
done
fi
du -sh $O
