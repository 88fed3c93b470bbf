cd $GRAFT_REPO_ROOT
O=gpurun_out/r02g; mkdir -p $O
timeout 600 python -m pytest tests/test_parity.py tests/test_capi.py -m gpu -x -q > $O/pytest.log 2>&1; echo pytest=$?; tail -2 $O/pytest.log
for cfg in C2 C3 T; do
  timeout 300 python scripts/po_profile.py $cfg 0 > $O/po_${cfg}_local.txt 2>&1
  timeout 300 python scripts/po_profile.py $cfg 8192 > $O/po_${cfg}_bsp.txt 2>&1
done
grep -h levels $O/po_*.txt
