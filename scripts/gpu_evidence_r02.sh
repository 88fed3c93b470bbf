# round-2 evidence: GPU tests, benches of every single-GPU config, launch
# lists and ncu --set full of T and C2 (raw / details / source pages exported
# on the box: gpurun brings back at most 64 MiB)
cd $GRAFT_REPO_ROOT
O=gpurun_out/${R:-r02ev}; mkdir -p $O
lscpu | grep -E "Model name|^CPU\(s\)" > $O/host.txt; free -g >> $O/host.txt
if [ -z "$NOTEST" ]; then timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo pytest=$?; tail -1 $O/pytest.log; fi
if [ -z "$NOBENCH" ]; then
timeout 1500 python bench.py > $O/bench_T.json 2> $O/bench_T.log; echo bench_T=$?
timeout 900 python bench.py --config C1 --steps 10 --extras "" > $O/bench_C1.json 2> $O/bench_C1.log; echo bench_C1=$?
timeout 1500 python bench.py --config C4 --steps 3 --extras "" > $O/bench_C4.json 2> $O/bench_C4.log; echo bench_C4=$?
grep "\[bench\]" $O/bench_*.log | grep -v graph | cut -c1-200
fi
if [ -z "$NONCU" ]; then
for cfg in C2 T; do
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"hc_|po_|rl_|DeviceScan" --csv --log-file $O/launches_${cfg}.csv python scripts/one_call.py $cfg > /dev/null 2>&1; echo launch_$cfg=$?
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"hc_rounds|hc_init|hc_el|po_levels|po_init|hc_degree|rl_arcs" -c 24 -o /tmp/prof_${cfg} python scripts/one_call.py $cfg > $O/ncu_$cfg.log 2>&1; echo ncu_$cfg=$?
  ncu -i /tmp/prof_${cfg}.ncu-rep --page raw --csv > $O/ncu_${cfg}_raw.csv 2>/dev/null
  ncu -i /tmp/prof_${cfg}.ncu-rep --page details --csv > $O/ncu_${cfg}_details.csv 2>/dev/null
  ncu -i /tmp/prof_${cfg}.ncu-rep --page source --csv --kernel-name regex:hc_rounds --launch-count 1 > $O/ncu_${cfg}_rounds_source.csv 2>/dev/null
  ncu -i /tmp/prof_${cfg}.ncu-rep --page source --csv --kernel-name regex:po_levels --launch-count 1 > $O/ncu_${cfg}_peel_source.csv 2>/dev/null
done
fi
du -sh $O
