cd $GRAFT_REPO_ROOT
cat > /tmp/chk.py <<'PY'
import sys, torch, numpy as np
sys.path.insert(0, '.')
import paper_2402_15253_b200 as pico, synth
cfg = sys.argv[1]; flags = int(sys.argv[2]) if len(sys.argv) > 2 else 0
rp, ci = synth.CONFIGS[cfg].build(device=torch.device("cuda:0"))
h = pico.coreness(rp, ci, algo="histocore")
for rep in range(2):
    st = pico.Stats()
    c = pico.coreness(rp, ci, algo="peelone", flags=flags, stats=st)
    bad = (c != h).sum().item()
    print(cfg, flags, "levels", st.levels, "kmax", st.kmax, "mismatch vs histocore", bad, flush=True)
PY
timeout 600 python -m pytest tests/test_parity.py tests/test_capi.py -m gpu -x -q 2>&1 | tail -1
for cfg in C2 C4 T; do timeout 300 python /tmp/chk.py $cfg; done
timeout 300 python /tmp/chk.py T 1024
for cfg in C2 C3 T; do timeout 300 python scripts/po_profile.py $cfg 0 2>&1 | grep -v "level sizes" | cut -c1-300; done
