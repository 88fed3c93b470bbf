#!/usr/bin/env python
"""Summarise ncu captures of one bench step into profiles/.

    python scripts/ncu_summary.py CONFIG ALGO REPORT.ncu-rep|RAW.csv [--out profiles/ncu_traffic.json]
    (ALGO is ignored: every kernel is keyed by the algorithm that launched it)
                                  [--md profiles/r01/ncu_CONFIG_ALGO.md]

Maps kernels to bench.py's kernel slots (degree / init / rounds / peel /
edgelist / relabel), sums dram__bytes_read.sum + dram__bytes_write.sum and
gpu__time_duration.sum per slot (one step = one launch of every slot kernel),
merges the per-slot DRAM bytes into the JSON that bench.py reports as
roofline.traffic, and writes a human-readable table of the key metrics.
"""
import csv
import io
import json
import subprocess
import sys

SLOTS = [
    ("rounds", ("hc_rounds_kernel",)),
    ("init", ("hc_init_small", "hc_init_warp", "hc_init_cta", "hc_init_fallback", "hc_shadow")),
    ("degree", ("hc_degree_kernel", "po_init_kernel")),
    ("peel", ("po_levels_kernel",)),
    ("edgelist", ("hc_el_",)),
    ("relabel", ("rl_bits", "rl_rows", "rl_pack", "rl_arcs", "rl_back", "DeviceScan")),
]
METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "lts__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
           "lts__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
           "lts__t_sectors_srcunit_tex_op_atom.sum", "lts__t_sectors_srcunit_tex_op_red.sum",
           "l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed"]
SCALE = {"gpu__time_duration.sum": {"ms": 1e-3, "us": 1e-6, "ns": 1e-9, "s": 1.0},
         "dram__bytes_read.sum": {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "Tbyte": 1e12},
         "dram__bytes_write.sum": {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "Tbyte": 1e12}}


def slot_of(name):
    for slot, keys in SLOTS:
        if any(k in name for k in keys):
            return slot
    return None


def main():
    cfg, algo, rep = sys.argv[1:4]
    out = "profiles/ncu_traffic.json"
    md = None
    if "--out" in sys.argv:
        out = sys.argv[sys.argv.index("--out") + 1]
    if "--md" in sys.argv:
        md = sys.argv[sys.argv.index("--md") + 1]
    if rep.endswith(".csv"):  # a raw page exported on the GPU box (ncu -i REP --page raw --csv)
        raw = open(rep).read()
    else:
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    # kernels are keyed by the algorithm whose call launched them: hc_* ->
    # histocore, po_* -> peelone; the shared compaction (rl_*, scans) belongs
    # to the call it runs in (scripts/one_call.py runs HistoCore first, then
    # PeelOne), i.e. its first launch to histocore, its second to peelone
    agg, lines, seen = {}, [], set()
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        name = d.get("Kernel Name", "")
        base = name.split("<")[0].split("(")[0].replace("void ", "").strip()
        if "hc_" in base:
            kalgo = "histocore"
        elif "po_" in base:
            kalgo = "peelone"
        else:
            kalgo = "histocore" if (base, "histocore") not in seen else "peelone"
        # one step = one launch of each distinct kernel per algorithm (the
        # bench's STATS run and timed runs use different template instances)
        if (base, kalgo) in seen:
            continue
        seen.add((base, kalgo))
        slot = slot_of(name)
        vals = {}
        for mtr in METRICS:
            try:
                v = float(d[mtr].replace(",", ""))
            except Exception:
                continue
            if v != v:  # nan (metric not collected for this launch)
                continue
            vals[mtr] = v * SCALE.get(mtr, {}).get(u.get(mtr, ""), 1.0)
        lines.append((name[:60], f"{kalgo}/{slot}", vals))
        if slot is None:
            continue
        a = agg.setdefault(kalgo, {}).setdefault(slot, {"dram_bytes_per_step": 0.0, "time_s": 0.0, "kernels": [],
                                                        "l2w": 0.0, "reqw": 0.0})
        a["dram_bytes_per_step"] += vals.get("dram__bytes_read.sum", 0) + vals.get("dram__bytes_write.sum", 0)
        a["time_s"] += vals.get("gpu__time_duration.sum", 0)
        # time-weighted L2 throughput (% of peak) of the slot's kernels: the second ceiling
        a["l2w"] += vals.get("lts__throughput.avg.pct_of_peak_sustained_elapsed", 0) * vals.get(
            "gpu__time_duration.sum", 0)
        # time-weighted busy share of the SM -> L2 request interface: the ceiling
        # a dense pull round hits (profiles/r02/s3/ncu_T_pull_rounds.md)
        a["reqw"] += vals.get("l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed", 0) * vals.get(
            "gpu__time_duration.sum", 0)
        a["kernels"].append(name[:60])
    try:
        with open(out) as f:
            allj = json.load(f)
    except Exception:
        allj = {}
    for kalgo, slots in agg.items():
        allj.setdefault(cfg, {})[kalgo] = {k: {"dram_bytes_per_step": v["dram_bytes_per_step"],
                                               "ncu_time_s": v["time_s"], "kernels": v["kernels"],
                                               "l2_throughput_pct": v["l2w"] / v["time_s"] if v["time_s"] else None,
                                               "l2_request_pct": v["reqw"] / v["time_s"] if v["time_s"] else None,
                                               "source": rep} for k, v in slots.items()}
    with open(out, "w") as f:
        json.dump(allj, f, indent=1, sort_keys=True)
    if md:
        with open(md, "w") as f:
            f.write(f"# ncu --set full summary: {cfg}, one HistoCore and one PeelOne call ({rep})\n\n")
            f.write("ncu replays each kernel with cold caches and serialised launches: times are for shares, "
                    "not absolutes.\n\n")
            f.write("| kernel | slot | time ms | DRAM read GB | DRAM write GB | L2 hit % | warps active % | L2 thru % | regs |\n")
            f.write("|---|---|---|---|---|---|---|---|---|\n")
            for name, slot, v in lines:
                f.write(f"| `{name}` | {slot} | {v.get('gpu__time_duration.sum', 0) * 1e3:.3f} | "
                        f"{v.get('dram__bytes_read.sum', 0) / 1e9:.3f} | {v.get('dram__bytes_write.sum', 0) / 1e9:.3f} | "
                        f"{v.get('lts__t_sector_hit_rate.pct', 0):.1f} | "
                        f"{v.get('sm__warps_active.avg.pct_of_peak_sustained_active', 0):.1f} | "
                        f"{v.get('lts__throughput.avg.pct_of_peak_sustained_elapsed', 0):.1f} | "
                        f"{v.get('launch__registers_per_thread', 0):.0f} |\n")
    print(json.dumps(allj[cfg], indent=1))


if __name__ == "__main__":
    main()
