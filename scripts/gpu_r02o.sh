cd $GRAFT_REPO_ROOT
O=gpurun_out/r02o; mkdir -p $O
timeout 900 python -m pytest tests/test_parity.py tests/test_dynamic.py -m gpu -x -q 2>&1 | tail -1
timeout 600 python scripts/round_profile.py --config T --reps 1 > $O/rp_T_e8.txt 2>&1
PICO_LIB=build_variants/libpico_e16.so timeout 600 python scripts/round_profile.py --config T --reps 1 > $O/rp_T_e16.txt 2>&1
head -1 $O/rp_T_e8.txt; tail -1 $O/rp_T_e8.txt; head -1 $O/rp_T_e16.txt; tail -1 $O/rp_T_e16.txt
