"""Aggregate ncu source-page stall samples (gpurun_out/source_<tag>.csv): totals per stall
reason and the top SASS lines by samples.  usage: python scripts/stalls.py TAG [top]"""
import csv
import sys

tag = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
rows = list(csv.reader(open(f"gpurun_out/source_{tag}.csv")))
hdr = rows[1]
si = hdr.index("Warp Stall Sampling (All Samples)")
ie = hdr.index("Instructions Executed")
stall_cols = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
tot = {h: 0 for _, h in stall_cols}
lines = []
all_s = 0
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    try:
        s = int(r[si])
    except ValueError:
        continue
    all_s += s
    for i, h in stall_cols:
        tot[h] += int(r[i] or 0)
    lines.append((s, r[1].strip(), r[ie]))
print(f"{tag}: {all_s} samples")
for h, v in sorted(tot.items(), key=lambda x: -x[1])[:10]:
    print(f"  {h:28s} {v:8d} {100.0 * v / max(all_s, 1):5.1f}%")
print("top lines:")
for s, src, ex in sorted(lines, reverse=True)[:top]:
    print(f"  {s:6d}  {ex:>8s}  {src[:90]}")
