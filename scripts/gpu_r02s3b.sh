# hub table: parity + T/C2 A/B (default vs PICO_F_NO_HUBS)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_parity.py tests/test_capi.py -m gpu -x -q 2>&1 | tail -3
for fl in 0 8192; do
  timeout 900 python bench.py --steps 3 --warmup 3 --no-oracle --extras C2 --no-both --flags $fl > gpurun_out/s3b_T_$fl.json 2> gpurun_out/s3b_T_$fl.log
  grep "histocore:" gpurun_out/s3b_T_$fl.log
done
timeout 900 python scripts/round_profile.py --config T --reps 1 > gpurun_out/s3b_rp_T.txt 2>&1; head -20 gpurun_out/s3b_rp_T.txt
timeout 1200 python -m pytest tests/test_fullsize.py -m gpu -x -q 2>&1 | tail -3
