"""Rank SASS instructions of an ncu report by executions and stall samples (development tool).

    ncu -i rep --page source --csv --print-source sass > sass.csv; python tools/ncu_sass_hot.py sass.csv
"""
import csv, sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ia, isrc, iex, ism = hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
data = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    try:
        data.append((int(r[ia], 16) if r[ia].startswith("0x") else int(r[ia]), r[isrc], float(r[iex] or 0), float(r[ism] or 0)))
    except ValueError:
        pass
tot = sum(d[2] for d in data)
tots = sum(d[3] for d in data)
print(f"total inst {tot:.3e}  samples {tots:.0f}")
# windows of 16 instructions
win = int(sys.argv[2]) if len(sys.argv) > 2 else 32
agg = []
for i in range(0, len(data), win):
    chunk = data[i:i + win]
    agg.append((sum(c[2] for c in chunk), sum(c[3] for c in chunk), chunk[0][0], chunk[0][1]))
for ex, sm, addr, src in sorted(agg, reverse=True)[:25]:
    print(f"{addr:#07x} inst {ex / tot * 100:5.1f}%  stall {sm / tots * 100:5.1f}%  {src[:60]}")
