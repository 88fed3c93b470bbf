# final code check: GPU tests, smoke, default bench, reference arm
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/s3final
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s3final/pytest.log 2>&1; echo pytest=$?; tail -1 gpurun_out/s3final/pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 1200 python bench.py > gpurun_out/s3final/bench_T.json 2> gpurun_out/s3final/bench_T.log; echo bench=$?
grep -E "histocore:|peelone:" gpurun_out/s3final/bench_T.log
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/s3final/bench_ref.json 2> gpurun_out/s3final/bench_ref.log; echo ref=$?
head -c 300 gpurun_out/s3final/bench_ref.json
