cd $GRAFT_REPO_ROOT
O=gpurun_out/r02r; mkdir -p $O
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=1 --master-addr 127.0.0.1 --master-port 29511 bench.py --sharded --config C1 --steps 3 --warmup 2 > $O/sh_C1.json 2> $O/sh_C1.log; echo c1=$?
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node=1 --master-addr 127.0.0.1 --master-port 29512 bench.py --sharded --config T --steps 3 --warmup 2 > $O/sh_T.json 2> $O/sh_T.log; echo t=$?
grep -h "bench-sharded\|NCCL INFO.*nranks\|Error\|error" $O/*.log | head -8
cat $O/sh_C1.json | head -c 1500; echo; cat $O/sh_T.json | head -c 2500
