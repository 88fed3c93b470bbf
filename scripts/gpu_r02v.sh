cd $GRAFT_REPO_ROOT
O=gpurun_out/r02v; mkdir -p $O
timeout 900 python -m pytest tests/test_parity.py tests/test_dynamic.py tests/test_fullsize.py -m gpu -x -q 2>&1 | tail -1
timeout 600 python scripts/round_profile.py --config T --reps 1 2>&1 | head -1 | cut -c1-250
timeout 600 python scripts/round_profile.py --config C4 --reps 1 2>&1 | head -1 | cut -c1-250
timeout 300 python scripts/po_profile.py C1 0 2>&1 | grep -v "level sizes" | cut -c1-400
