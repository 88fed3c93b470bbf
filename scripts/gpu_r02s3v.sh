# stress before committing the entry encoding: GPU tests + 10 bounded rounds of every config
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
sed -n '/^cat > \/tmp\/po_ab.py/,/^PY$/p' scripts/gpu_r02s3h.sh | sed '1d;$d' > /tmp/po_ab.py
for rep in 1 2 3 4 5 6 7 8 9 10; do
  t0=$(date +%s)
  timeout 240 python /tmp/po_ab.py C1 C2 C3 T C4 > /tmp/o.txt 2>&1
  echo "rep $rep rc=$? $(( $(date +%s) - t0 ))s $(tail -1 /tmp/o.txt | cut -c1-200)"
done
