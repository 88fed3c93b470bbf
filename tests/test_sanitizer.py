"""compute-sanitizer memcheck / racecheck / synccheck over every
kernel family of libpico on small graphs (HistoCore push / pull / host loop /
debug check, PeelOne, CntCore, NbrCore, the sharded HistoCore and PeelOne kernels in loopback,
the decremental update and an insertion)."""
import os
import re
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys, torch
sys.path.insert(0, %r)
import synth, paper_2402_15253_b200 as pico
from paper_2402_15253_b200 import sharded
rp, ci = synth.CONFIGS["R12"].build(device=torch.device("cuda:0"))
for algo, fl in (("histocore", 0), ("histocore", pico.F_PULL_ALWAYS | pico.F_TINY_TILES),
                 ("histocore", pico.F_HOST_LOOP | pico.F_DEBUG_INVARIANTS), ("peelone", 0),
                 ("peelone", pico.F_CLAMP_CAS), ("cntcore", 0), ("nbrcore", 0), ("auto", pico.F_VALIDATE)):
    pico.coreness(rp, ci, algo=algo, flags=fl)
if %r:
    sharded.coreness_loopback(rp, ci, 3, pico.F_PULL_ALWAYS)
    sharded.coreness_loopback_peel(rp, ci, 3, pico.F_TINY_TILES)
    d = pico.DynamicCoreness(rp, ci)
    src = torch.repeat_interleave(torch.arange(rp.numel() - 1, device=rp.device), rp[1:] - rp[:-1])
    m = src < ci
    d.delete_edges(src[m][:50].int(), ci[m][:50])
    d.insert_edges(src[m][:50].int(), ci[m][:50])  # the same edges back: insertion path
    d.coreness()
    d.close()
torch.cuda.synchronize()
print("done")
"""


def _sanitize(tool, full):
    cs = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    if not os.path.exists(cs):
        pytest.skip("compute-sanitizer not found")
    cmd = [cs, "--tool", tool, "--error-exitcode", "3", sys.executable, "-c", SCRIPT % (ROOT, full)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1200)
    out = r.stdout + r.stderr
    if "done" not in out and ("closed on this pool" in out or "is closed" in out):
        # the GPU pool's compute-sanitizer wrapper refuses to run (not a kernel error)
        pytest.skip("compute-sanitizer unavailable on this GPU pool: " + out.strip()[:200])
    assert r.returncode == 0 and "done" in out, out[-4000:]
    # memcheck / synccheck: "ERROR SUMMARY: 0 errors"; racecheck: "RACECHECK SUMMARY: 0 hazards displayed (0 errors, 0 warnings)"
    counts = [int(x) for x in re.findall(r"SUMMARY: (\d+) (?:errors|hazards)", out)]
    assert counts and not any(counts), out[-4000:]
    assert "(0 errors" in out or tool != "racecheck", out[-4000:]


def test_memcheck():
    _sanitize("memcheck", True)


@pytest.mark.parametrize("tool", ["racecheck", "synccheck"])
def test_race_and_sync(tool):
    _sanitize(tool, False)
