# evidence at the PeelOne barrier/queue change: GPU tests, default bench (T + C2/C3), C4/C1 benches
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/s3n
timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 | tee gpurun_out/s3n/pytest_summary.txt
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/s3n/bench_T.json 2> gpurun_out/s3n/bench_T.log
grep -E "histocore:|peelone:" gpurun_out/s3n/bench_T.log
for cfg in C4 C1; do
  timeout 900 python bench.py --config $cfg --steps 5 --warmup 3 --extras '' > gpurun_out/s3n/bench_$cfg.json 2> gpurun_out/s3n/bench_$cfg.log
  grep -E "histocore:|peelone:" gpurun_out/s3n/bench_$cfg.log
done
