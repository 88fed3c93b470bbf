# LSA device exchange with the cached window: one-rank tests + sharded bench C2/T A/B
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export NCCL_DEBUG=WARN
timeout 900 python -m pytest tests/test_sharded.py -m gpu -x -q -k "lsa or single_rank_nccl" 2>&1 | tail -2
for run in "nccl 4" "lsa 4" "lsa 8" "lsa 2"; do
  set -- $run
  for cfg in C2 T; do
    PICO_LSA_BATCH=$2 timeout 900 torchrun --nnodes 1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --sharded --config $cfg --steps 5 --warmup 3 --exchange $1 > gpurun_out/s3e_sh_${cfg}_$1_$2.json 2> gpurun_out/s3e_sh_${cfg}_$1_$2.log
    python -c "
import json; d=json.load(open('gpurun_out/s3e_sh_${cfg}_$1_$2.json')); print('$cfg $1 batch $2', d['ms_per_step'])" 2>&1 | tail -1
  done
done
