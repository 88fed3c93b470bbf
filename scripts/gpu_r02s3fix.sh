# near/far rebuild loop: the 1.5k+16 rule that failed now, and the default, over 117 RMAT graphs; parity
cd $GRAFT_REPO_ROOT
for v in fix15 fix2; do echo "== $v"; PICO_LIB=build_variants/libpico_$v.so timeout 800 python scripts/peel_find.py 2>&1 | grep -E "FAIL|scale 24" | head -5; done
timeout 900 python -m pytest tests/test_parity.py tests/test_fullsize.py -m gpu -x -q 2>&1 | tail -1
sed -n '/^cat > \/tmp\/po_ab.py/,/^PY$/p' scripts/gpu_r02s3h.sh | sed '1d;$d' > /tmp/po_ab.py
for v in fix2 fix15 w2a16; do PICO_LIB=build_variants/libpico_$v.so timeout 300 python /tmp/po_ab.py C2 C3 T C4 2>&1 | tail -1 | sed 's/"histocore": [0-9.]*//g'; done
