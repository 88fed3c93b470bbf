# flip-word grid barrier + two PeelOne queue logs: parity, full size, benches
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_parity.py tests/test_capi.py -m gpu -x -q 2>&1 | tail -2
timeout 900 python bench.py --steps 5 --warmup 3 --no-oracle --extras C2,C3 > gpurun_out/s3f_T.json 2> gpurun_out/s3f_T.log
grep -E "histocore:|peelone:" gpurun_out/s3f_T.log
timeout 900 python scripts/po_profile.py --config C2 > gpurun_out/s3f_po_C2.txt 2>&1; head -4 gpurun_out/s3f_po_C2.txt | cut -c1-300
timeout 1500 python -m pytest tests/test_fullsize.py tests/test_sanitizer.py -m gpu -x -q 2>&1 | tail -2
