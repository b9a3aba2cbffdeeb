"""Per-region (BAR.SYNC-delimited) stall and instruction-mix breakdown of an
`ncu --page source --csv --print-source sass` export (first kernel section).
    python tools/sass_regions.py file.csv"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
cut = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"]
if len(cut) > 1:
    rows = rows[: cut[1]]
hdr = rows[1]
data = [r for r in rows[2:] if len(r) == len(hdr) and r[0].startswith("0x")]
ix = {h: i for i, h in enumerate(hdr)}
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
reg, agg, cnt = 0, {}, {}
for r in data:
    src = r[ix["Source"]].strip()
    d = agg.setdefault(reg, {})
    for s in stalls:
        d[s] = d.get(s, 0) + int(r[ix[s]] or 0)
    op = (src.split()[1] if src.startswith("@") else src.split()[0]).split(".")[0]
    c = cnt.setdefault(reg, {})
    c[op] = c.get(op, 0) + int(r[ix["Instructions Executed"]] or 0)
    if "BAR.SYNC" in src:
        reg += 1
T = sum(sum(d.values()) for d in agg.values())
I = sum(sum(c.values()) for c in cnt.values())
print(f"total warp-instructions {I}")
for k, d in agg.items():
    t = sum(d.values())
    n = sum(cnt[k].values())
    print(f"region {k}: {100*t/T:.0f}% of samples, {100*n/I:.0f}% of instructions ({n}); stalls: "
          + ", ".join(f"{s[6:]} {100*v/max(t,1):.0f}%" for s, v in sorted(d.items(), key=lambda x: -x[1])[:5]))
    print("    mix:", ", ".join(f"{o} {v}" for o, v in sorted(cnt[k].items(), key=lambda x: -x[1])[:10]))
