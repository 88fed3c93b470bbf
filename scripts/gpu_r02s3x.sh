# NVTX phase ranges: ncu filtered by range sees only that phase's kernels; one-rank LSA sanity
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/s3x
for r in rounds peel init edgelist; do
  timeout 300 ncu --nvtx --nvtx-include "pico:$r/" --metrics gpu__time_duration.sum --csv python scripts/one_call.py C2 > gpurun_out/s3x/nvtx_$r.csv 2>/dev/null
  python -c "import csv;rows=[r for r in csv.reader(open('gpurun_out/s3x/nvtx_$r.csv')) if len(r)>10 and r[0].isdigit()];print('$r',sorted(set(x[6].split('(')[0] for x in rows)))"
done
