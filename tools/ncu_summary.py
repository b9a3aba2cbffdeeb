"""Summarise ncu outputs into profiles/ (tracked evidence).

    python tools/ncu_summary.py <tag> <launches.csv> <full.ncu-rep[,more.ncu-rep]> <pairs> [launch-list command]

Writes profiles/<tag>_launches.md (per-kernel share of a registration, cold-cache
serialised ncu times: compare SHARES, not absolutes), profiles/<tag>_ncu_full.md
(key metrics + stall reasons of the captured kernels) and profiles/xpass_dram_bytes.json
(DRAM bytes of one x-pass launch, read by bench.py for roofline.traffic).
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.environ.get("DREG_PROF_DIR") or os.path.join(ROOT, "profiles")


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hdr_i]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[hdr_i + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0].replace("void ", "")
        agg[name][0] += 1
        agg[name][1] += float(r[vi].replace(",", ""))
    return agg


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def main():
    tag, lcsv, rep, pairs = sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4])
    cmd = sys.argv[5] if len(sys.argv) > 5 else None
    os.makedirs(PROF, exist_ok=True)
    agg = launches(lcsv)
    tot = sum(v[1] for v in agg.values())
    lines = [f"# {tag}: ncu launch list (`--metrics gpu__time_duration.sum --clock-control none`)", "",
             (f"Command: `{cmd}`." if cmd else
              f"Command: `python tools/profile_step.py {pairs} 1` (one registration chunk of {pairs} config-2 pairs, "
              "1 velocity field x 50 iterations, then the per-kernel timing loop).") +
             "  ncu serialises launches and runs them cold-cache: use the SHARES.", "",
             "| kernel | launches | total us | share |", "|---|---|---|---|"]
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| `{k}` | {n} | {t / 1e3:.1f} | {100 * t / tot:.1f}% |")
    open(os.path.join(PROF, f"{tag}_launches.md"), "w").write("\n".join(lines) + "\n")

    reps = rep.split(",")
    hdr, _, _ = raw(reps[0])
    data, units_of = [], []
    for r_ in reps:  # every capture keeps its own units row
        h2, u2, d2 = raw(r_)
        for row in d2:
            data.append([row[h2.index(h)] if h in h2 else "" for h in hdr])
            units_of.append([u2[h2.index(h)] if h in h2 else "" for h in hdr])
    want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
            "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers", "smsp__inst_executed.sum",
            "smsp__issue_active.avg.pct_of_peak_sustained_active", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
            "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"]
    out = [f"# {tag}: ncu --set full (`--clock-control none`) of the per-iteration kernels", "",
           f"Captured from `python tools/profile_step.py {pairs} 1`; {pairs} config-2 pairs per launch "
           "(dram bytes are per launch).", ""]
    dram = {}
    for r, units in zip(data, units_of):
        name = r[hdr.index("Kernel Name")]
        out.append(f"## `{name}`")
        out.append("")
        out.append("| metric | value | unit |")
        out.append("|---|---|---|")
        for w in want:
            if w in hdr:
                i = hdr.index(w)
                out.append(f"| {w} | {r[i]} | {units[i]} |")
        stalls = []
        for i, h in enumerate(hdr):
            if "smsp__pcsamp_warps_issue_stalled" in h and not h.endswith("not_issued"):
                try:
                    stalls.append((float(r[i]), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        s = sum(v for v, _ in stalls) or 1.0
        out.append("")
        out.append("stall reasons: " + ", ".join(f"{h} {100 * v / s:.0f}%" for v, h in sorted(stalls, reverse=True)[:8]))
        out.append("")
        if "xpass" in name and "dram__bytes_read.sum" in hdr:
            def b(w):
                i = hdr.index(w)
                v = float(r[i].replace(",", ""))
                u = units[i]
                return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(u, 1)
            dram = {"kernel": name, "dram_bytes_per_launch": b("dram__bytes_read.sum") + b("dram__bytes_write.sum"),
                    "pairs": pairs, "source": f"profiles/{tag}_ncu_full.md"}
    open(os.path.join(PROF, f"{tag}_ncu_full.md"), "w").write("\n".join(out) + "\n")
    if dram:
        json.dump(dram, open(os.path.join(PROF, "xpass_dram_bytes.json"), "w"), indent=1)
    print("wrote", tag)


if __name__ == "__main__":
    main()
