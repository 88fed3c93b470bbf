"""Top stall instructions and memory instructions of one kernel in an ncu
report (source page, SASS).  usage: ncu_source.py report.ncu-rep [kernel-regex] [top]"""
import csv
import subprocess
import sys


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


def main(path, kern="hc_", top=25):
    out = subprocess.check_output(["ncu", "-i", path, "--page", "source", "--csv", "--kernel-name",
                                   "regex:" + kern, "--launch-count", "1"], text=True)
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[1]
    ci = {h: i for i, h in enumerate(hdr)}
    data = [r for r in rows[2:] if len(r) == len(hdr) and r[0] != "Address"]
    seen, uniq = set(), []
    for r in data:
        if r[ci["Address"]] in seen:
            continue
        seen.add(r[ci["Address"]])
        uniq.append(r)
    K = "Warp Stall Sampling (All Samples)"
    tot = sum(f(r[ci[K]]) for r in uniq) or 1
    print(f"samples {tot:.0f}")
    stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    agg = {h: sum(f(r[ci[h]]) for r in uniq) for h in stalls}
    print("stall mix:", ", ".join(f"{k[6:]} {v / tot * 100:.1f}%" for k, v in sorted(agg.items(), key=lambda x: -x[1])[:8]))
    for r in sorted(uniq, key=lambda r: -f(r[ci[K]]))[:top]:
        s = f(r[ci[K]])
        main_stall = max(stalls, key=lambda h: f(r[ci[h]]))
        print(f"{s / tot * 100:5.1f}% {r[ci['Address']][-5:]} {r[ci['Source']][:64]:64} [{main_stall[6:]}]")


if __name__ == "__main__":
    main(sys.argv[1], *(sys.argv[2:3] or []), *(int(x) for x in sys.argv[3:4]))
