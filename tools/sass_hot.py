"""Summarise an `ncu --page source --csv --print-source sass` export: stall totals by
reason and by kernel region (split at BAR.SYNC), plus the hottest instructions.
    python tools/sass_hot.py file.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
cut = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"]
if len(cut) > 1:
    rows = rows[: cut[1]]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
hdr = rows[1]
data = [r for r in rows[2:] if len(r) == len(hdr) and r[0].startswith("0x")]  # first kernel section
ix = {h: i for i, h in enumerate(hdr)}
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = {s: 0 for s in stalls}
region, regions = 0, {}
for r in data:
    src = r[ix["Source"]].strip()
    n = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    regions.setdefault(region, [0, src])[0] += n
    for s in stalls:
        tot[s] += int(r[ix[s]] or 0)
    if "BAR.SYNC" in src or "BAR.SYNC.DEFER_BLOCKING" in src:
        region += 1
T = sum(tot.values())
print("stalls:", ", ".join(f"{k[6:]} {100*v/T:.0f}%" for k, v in sorted(tot.items(), key=lambda x: -x[1]) if v))
print("samples per barrier-delimited region:", {k: f"{100*v[0]/T:.0f}%" for k, v in regions.items()})
hot = sorted(data, key=lambda r: -int(r[ix["Warp Stall Sampling (All Samples)"]] or 0))[:top]
for r in hot:
    n = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    why = sorted(((int(r[ix[s]] or 0), s[6:]) for s in stalls), reverse=True)[:2]
    print(f"{100*n/T:5.1f}% {r[ix['Address']][-5:]} {r[ix['Source']].strip()[:60]:60s} {why}")
