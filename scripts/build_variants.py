"""Build A/B variants of libpico.so under build_variants/ (git-ignored; they
travel to the GPU box with gpurun).  usage: python scripts/build_variants.py name=DEF1,DEF2 ..."""
import os
import sys
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2402_15253_b200 import build as b  # noqa: E402

os.makedirs(os.path.join(b.ROOT, "build_variants"), exist_ok=True)


def one(spec):
    name, _, defs = spec.partition("=")
    out = os.path.join(b.ROOT, "build_variants", f"libpico_{name}.so")
    b.build(force=True, out=out, defines=[d for d in defs.split(",") if d])
    return out


with ThreadPoolExecutor(4) as ex:
    for o in ex.map(one, sys.argv[1:]):
        print(o)
