# sharded PeelOne with the device-driven level loop (LSA): one-rank tests + C2/T A/B vs the host exchange
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export NCCL_DEBUG=WARN
timeout 900 python -m pytest tests/test_sharded.py -m gpu -x -q -k "lsa or single_rank_nccl" 2>&1 | tail -4
for ex in nccl lsa; do
  for cfg in C2 T; do
    timeout 900 torchrun --nnodes 1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --sharded --algo peelone --config $cfg --steps 5 --warmup 3 --exchange $ex > gpurun_out/s3q_shpo_${cfg}_$ex.json 2> gpurun_out/s3q_shpo_${cfg}_$ex.log
    python -c "
import json; d=json.load(open('gpurun_out/s3q_shpo_${cfg}_$ex.json')); print('$cfg peel $ex', d['ms_per_step'])" 2>&1 | tail -1
  done
done
