cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_parity.py tests/test_sharded.py tests/test_dynamic.py -m gpu -x -q 2>&1 | tail -1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"hc_init" --csv python scripts/one_call.py T histocore 2>/dev/null | grep -o '"pico::[^"]*hc_init[^"]*\|"void pico::hc_init[^"]*\|"[0-9,.]*"$' | paste - - 
