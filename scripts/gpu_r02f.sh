cd $GRAFT_REPO_ROOT
O=gpurun_out/r02f; mkdir -p $O
timeout 300 python -m pytest tests/test_parity.py -m gpu -x -q -k "peel or corpus or fixture" > $O/pytest.log 2>&1; echo pytest=$?; tail -2 $O/pytest.log
timeout 240 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"po_" --csv --log-file $O/launches_C1_po.csv python scripts/one_call.py C1 peelone > $O/ncu_c1.log 2>&1; echo launch_C1=$?
timeout 400 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"po_" --csv --log-file $O/launches_T_po.csv python scripts/one_call.py T peelone > $O/ncu_T.log 2>&1; echo launch_T=$?
tail -3 $O/ncu_T.log
