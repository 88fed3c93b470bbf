# final code: the driver's default bench three times, then the GPU tests
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/s3ev4
for i in 1 2 3; do
  timeout 1200 python bench.py > gpurun_out/s3ev4/bench_T_$i.json 2> gpurun_out/s3ev4/bench_T_$i.log; echo bench_$i=$?
  grep -E "histocore:|peelone:|Error|error" gpurun_out/s3ev4/bench_T_$i.log | cut -c1-110
done
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
