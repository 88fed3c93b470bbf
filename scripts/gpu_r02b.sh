cd $GRAFT_REPO_ROOT
O=gpurun_out/r02b; mkdir -p $O
timeout 600 python scripts/round_profile.py --config T --reps 2 > $O/rp_T_default.txt 2>&1
timeout 600 python scripts/round_profile.py --config T --reps 1 --flags 64 > $O/rp_T_push.txt 2>&1
timeout 600 python scripts/round_profile.py --config T --reps 1 --flags 128 > $O/rp_T_pull.txt 2>&1
