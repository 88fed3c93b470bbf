cd $GRAFT_REPO_ROOT
O=gpurun_out/r02c; mkdir -p $O
timeout 900 python -m pytest tests/test_parity.py tests/test_capi.py tests/test_dynamic.py -m gpu -x -q > $O/pytest.log 2>&1; echo pytest=$?; tail -3 $O/pytest.log
timeout 600 python scripts/round_profile.py --config T --reps 1 > $O/rp_T_default.txt 2>&1
timeout 600 python scripts/round_profile.py --config T --reps 1 --flags 128 > $O/rp_T_pull.txt 2>&1
timeout 600 python scripts/round_profile.py --config C2 --reps 2 --flags 128 > $O/rp_C2_pull.txt 2>&1
timeout 600 python scripts/round_profile.py --config C2 --reps 2 > $O/rp_C2_default.txt 2>&1
