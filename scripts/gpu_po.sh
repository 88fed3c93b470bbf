cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for fl in 0 16 1024; do
timeout 600 python bench.py --steps 5 --warmup 3 --no-oracle --no-both --algo peelone --flags $fl > gpurun_out/po_$fl.json 2>/dev/null
python -c "
import json;d=json.load(open('gpurun_out/po_$fl.json'));r=d['per_algo']['peelone']
print('C2 flags $fl ms %.2f'%r['ms'], r['kernel_ms_per_step'])"
done
timeout 900 python bench.py --config T --steps 3 --warmup 3 --no-oracle --no-both --algo peelone > gpurun_out/po_T.json 2>/dev/null
python -c "
import json;d=json.load(open('gpurun_out/po_T.json'));r=d['per_algo']['peelone']
print('T ms %.2f'%r['ms'], r['kernel_ms_per_step'])"
