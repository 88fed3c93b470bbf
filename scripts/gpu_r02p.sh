cd $GRAFT_REPO_ROOT
O=gpurun_out/r02p; mkdir -p $O
timeout 900 python -m pytest tests/test_parity.py -m gpu -x -q -k "histocore or corpus or fixture or rmat" 2>&1 | tail -1
PICO_LIB=build_variants/libpico_vec.so timeout 900 python -m pytest tests/test_parity.py -m gpu -x -q -k "histocore or corpus or rmat" 2>&1 | tail -1
timeout 600 python scripts/round_profile.py --config T --reps 1 > $O/rp_T_base.txt 2>&1
timeout 600 python scripts/round_profile.py --config T --reps 1 --flags 16384 > $O/rp_T_persist.txt 2>&1
PICO_LIB=build_variants/libpico_vec.so timeout 600 python scripts/round_profile.py --config T --reps 1 > $O/rp_T_vec.txt 2>&1
for f in base persist vec; do echo $f; head -1 $O/rp_T_$f.txt | cut -c1-200; tail -1 $O/rp_T_$f.txt; done
