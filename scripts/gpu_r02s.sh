cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_dynamic.py tests/test_capi.py -m gpu -x -q 2>&1 | tail -15
