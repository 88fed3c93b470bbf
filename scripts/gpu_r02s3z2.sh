# PeelOne initial near window (PICO_PO_KHI0) sweep, same box
cd $GRAFT_REPO_ROOT
sed -n '/^cat > \/tmp\/po_ab.py/,/^PY$/p' scripts/gpu_r02s3h.sh | sed '1d;$d' > /tmp/po_ab.py
for rep in 1 2; do
for v in w2a16 w2a8 w15a16 w3a16 w2a32; do
  PICO_LIB=build_variants/libpico_$v.so timeout 300 python /tmp/po_ab.py C2 C3 T C4 2>&1 | tail -1 | sed 's/"histocore": [0-9.]*//g'
done
done
