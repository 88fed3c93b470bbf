cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_parity.py tests/test_capi.py tests/test_fullsize.py -m gpu -x -q 2>&1 | tail -1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 2>/dev/null | head -c 600; echo
