# LSA device exchange: one-rank tests + sharded bench C2/T (host exchange vs LSA); T NO_RELABEL A/B
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export NCCL_DEBUG=WARN
timeout 900 python -m pytest tests/test_sharded.py -m gpu -x -q -k "lsa or single_rank_nccl" 2>&1 | tail -5
for ex in nccl lsa; do
  for cfg in C2 T; do
    timeout 900 torchrun --nnodes 1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --sharded --config $cfg --steps 5 --warmup 3 --exchange $ex > gpurun_out/s3d_sh_${cfg}_$ex.json 2> gpurun_out/s3d_sh_${cfg}_$ex.log
    python -c "
import json; d=json.load(open('gpurun_out/s3d_sh_${cfg}_$ex.json')); print('$cfg $ex', d['ms_per_step'], d['config'].get('parallelism'))" 2>&1 | tail -1
  done
done
timeout 900 python bench.py --steps 3 --warmup 3 --no-oracle --extras '' --no-both --flags 512 > gpurun_out/s3d_T_norelabel.json 2> gpurun_out/s3d_T_norelabel.log; grep "histocore:" gpurun_out/s3d_T_norelabel.log
