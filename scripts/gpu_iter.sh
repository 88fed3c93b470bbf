# iteration script: GPU tests + C2 bench + T bench (no oracle)
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.log; echo rc=$?
grep "\[bench\]" gpurun_out/bench_c2.log | tail -4
python -c "import json;d=json.load(open('gpurun_out/bench_c2.json'));print('C2 value',d['value']/1e9,'ms',d['ms_per_step'],'frac',d['roofline']['frac'],'e2e',d['e2e']['ms_per_step'],'parity',d['parity'],'cpu',d['cpu_baseline'])"
timeout 900 python bench.py --config T --steps 3 --warmup 3 --no-oracle > gpurun_out/bench_T.json 2> gpurun_out/bench_T.log; echo rcT=$?
grep "\[bench\]" gpurun_out/bench_T.log | tail -4; tail -2 gpurun_out/bench_T.log
