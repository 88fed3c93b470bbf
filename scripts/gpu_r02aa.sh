cd $GRAFT_REPO_ROOT
PICO_LIB=build_variants/libpico_nored.so timeout 600 python scripts/round_profile.py --config T --reps 1 2>&1 > gpurun_out/rp_nored.txt
timeout 600 python scripts/round_profile.py --config T --reps 1 2>&1 > gpurun_out/rp_base.txt
paste <(sed -n 3,50p gpurun_out/rp_base.txt | awk '{print $1, $4, $5}') <(sed -n 3,50p gpurun_out/rp_nored.txt | awk '{print $2, $5}') | head -48
