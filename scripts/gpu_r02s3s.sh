# PeelOne queue entries holding their arc range (no row-bound loads in the drain): parity + A/B
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity.py tests/test_capi.py -m gpu -x -q 2>&1 | tail -1
sed -n '/^cat > \/tmp\/po_ab.py/,/^PY$/p' scripts/gpu_r02s3h.sh | sed '1d;$d' > /tmp/po_ab.py
for rep in 1 2; do
for v in cur enc; do
  PICO_LIB=build_variants/libpico_$v.so timeout 600 python /tmp/po_ab.py C1 C2 C3 T C4 2>&1 | tail -1
done
done
