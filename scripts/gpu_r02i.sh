cd $GRAFT_REPO_ROOT
O=gpurun_out/r02i; mkdir -p $O
timeout 600 python -m pytest tests/test_parity.py tests/test_capi.py -m gpu -x -q > $O/pytest.log 2>&1; echo pytest=$?; tail -1 $O/pytest.log
for cfg in C2 C3 T; do timeout 300 python scripts/po_profile.py $cfg 0 2>&1 | grep -v "^level sizes" | tee $O/po_$cfg.txt; done
