# Fig 3 frontier counts: parity test + bench lines with the fig3 summary
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/s3p
timeout 1200 python -m pytest tests/test_parity.py tests/test_capi.py -m gpu -x -q 2>&1 | tail -3
timeout 900 python bench.py --steps 5 --warmup 3 --extras C2,C3 > gpurun_out/s3p/bench_T.json 2> gpurun_out/s3p/bench_T.log
grep -E "histocore:|peelone:|parity" gpurun_out/s3p/bench_T.log | head
python -c "
import json; d=json.load(open('gpurun_out/s3p/bench_T.json'))
print('T fig3', d['per_algo']['histocore'].get('fig3'))
for c,v in d.get('per_config',{}).items(): print(c, 'fig3', v['per_algo']['histocore'].get('fig3'))
" 2>&1 | tail -4
