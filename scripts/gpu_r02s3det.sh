cd $GRAFT_REPO_ROOT
for v in w15a16 w2a16; do PICO_LIB=build_variants/libpico_$v.so timeout 300 python scripts/peel_det.py; done
timeout 300 python scripts/peel_det.py
