cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=1 --master-addr 127.0.0.1 --master-port 29611 bench.py --sharded --steps 5 --warmup 3 > gpurun_out/bench_c2_shard1.json 2> gpurun_out/bench_c2_shard1.log; echo rc=$?
python -c "
import json;d=json.load(open('gpurun_out/bench_c2_shard1.json')); print('sharded P=1 C2 ms %.2f'%d['ms_per_step'], 'e2e %.1f'%d['e2e']['ms_per_step'], d['parity'])"
