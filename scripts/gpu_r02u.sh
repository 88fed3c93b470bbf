cd $GRAFT_REPO_ROOT
O=gpurun_out/r02u; mkdir -p $O
PICO_LIB=build_variants/libpico_l1.so timeout 900 python -m pytest tests/test_parity.py -m gpu -x -q -k "histocore or corpus or rmat" 2>&1 | tail -1
timeout 600 python scripts/round_profile.py --config T --reps 1 > $O/rp_T.txt 2>&1
PICO_LIB=build_variants/libpico_l1.so timeout 600 python scripts/round_profile.py --config T --reps 1 > $O/rp_T_l1.txt 2>&1
head -1 $O/rp_T.txt | cut -c1-220; tail -1 $O/rp_T.txt; head -1 $O/rp_T_l1.txt | cut -c1-220; tail -1 $O/rp_T_l1.txt
