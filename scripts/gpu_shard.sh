cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=1 --master-addr 127.0.0.1 --master-port 29611 bench.py --sharded --steps 5 --warmup 3 > gpurun_out/bench_c2_shard1.json 2> gpurun_out/bench_c2_shard1.log; echo rc=$?
tail -c 1500 gpurun_out/bench_c2_shard1.json; tail -3 gpurun_out/bench_c2_shard1.log
