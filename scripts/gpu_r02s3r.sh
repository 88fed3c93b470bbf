# PeelOne light sub-rounds: degree prefetch A/B (threshold 0 = off, 4096, 65536), same box
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity.py -m gpu -x -q -k "peelone or c1 or fixtures" 2>&1 | tail -1
sed -n '/^cat > \/tmp\/po_ab.py/,/^PY$/p' scripts/gpu_r02s3h.sh | sed '1d;$d' > /tmp/po_ab.py
for rep in 1 2; do
for v in light0 light light64k; do
  PICO_LIB=build_variants/libpico_$v.so timeout 600 python /tmp/po_ab.py C1 C2 C3 T 2>&1 | tail -1
done
done
