# the level-head race fix: stress (15 bounded rounds of every config) + parity
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_parity.py tests/test_capi.py -m gpu -x -q 2>&1 | tail -1
sed -n '/^cat > \/tmp\/po_ab.py/,/^PY$/p' scripts/gpu_r02s3h.sh | sed '1d;$d' > /tmp/po_ab.py
for rep in $(seq 1 15); do
  t0=$(date +%s)
  timeout 200 python /tmp/po_ab.py C1 C2 C3 T C4 > /tmp/o.txt 2>&1
  echo "rep $rep rc=$? $(( $(date +%s) - t0 ))s $(tail -1 /tmp/o.txt | cut -c1-220)"
done
