# PeelOne barrier A/B on one box: base (HEAD~: one log + snapshot barrier), flip (two logs + flip-word
# barrier), flip32 (+32 ns poll backoff), gen (two logs + the generation-word barrier)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
cat > /tmp/po_ab.py <<'PY'
import os, sys, time, json
import torch
sys.path.insert(0, os.getcwd())
import paper_2402_15253_b200 as pico, synth
res = {}
for cfg in sys.argv[1:]:
    rp, ci = synth.CONFIGS[cfg].build(device=torch.device("cuda:0"))
    torch.cuda.synchronize(); torch.cuda.empty_cache()
    out = {}
    for algo in ("peelone", "histocore"):
        for _ in range(3): pico.coreness(rp, ci, algo=algo)
        torch.cuda.synchronize()
        reps = 10 if cfg != "T" else 4
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps): pico.coreness(rp, ci, algo=algo)
        e1.record(); torch.cuda.synchronize()
        out[algo] = round(e0.elapsed_time(e1) / reps, 3)
    res[cfg] = out
    del rp, ci; torch.cuda.empty_cache()
print(os.environ.get("PICO_LIB", "default").split("/")[-1], json.dumps(res))
PY
for rep in 1 2; do
for v in base flip flip32 gen; do
  PICO_LIB=build_variants/libpico_$v.so timeout 600 python /tmp/po_ab.py C2 C3 T 2>&1 | tail -1
done
done
