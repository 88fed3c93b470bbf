# single-log snapshot-free queue + flip barrier: parity + A/B vs base/gen
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_parity.py tests/test_capi.py -m gpu -x -q 2>&1 | tail -2
sed -n '/^cat > \/tmp\/po_ab.py/,/^PY$/p' scripts/gpu_r02s3h.sh | sed '1d;$d' > /tmp/po_ab.py
for rep in 1 2; do
for v in base flip gen; do
  PICO_LIB=build_variants/libpico_$v.so timeout 600 python /tmp/po_ab.py C2 C3 T 2>&1 | tail -1
done
done
