# session 3 of round 2: state check + hub/smem microbenchmarks
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
./scripts/micro/smem_gather > gpurun_out/smem_gather.txt 2>&1
timeout 600 python scripts/hub_share.py T C4 C2 > gpurun_out/hub_share.txt 2>&1
timeout 900 python bench.py --steps 3 --warmup 3 --no-oracle --extras C2 > gpurun_out/s3a_T.json 2> gpurun_out/s3a_T.log
tail -3 gpurun_out/s3a_T.log
cat gpurun_out/smem_gather.txt gpurun_out/hub_share.txt
