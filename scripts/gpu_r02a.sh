cd $GRAFT_REPO_ROOT
O=gpurun_out/r02a; mkdir -p $O
nproc > $O/host.txt; free -g >> $O/host.txt
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo pytest=$?; tail -3 $O/pytest.log
timeout 1200 python bench.py > $O/bench_default.json 2> $O/bench_default.log; echo bench=$?
tail -5 $O/bench_default.log
