"""Hottest SASS instructions of an ncu source capture with their stall reasons.

    ncu -i REP --page source --csv --print-source sass > x.csv
    python tools/sass_hot.py x.csv [top] [context]
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
ctx = int(sys.argv[3]) if len(sys.argv) > 3 else 0
hdr = rows[1]
ia, isrc = hdr.index("Address"), hdr.index("Source")
isamp, iexe = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
reasons = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
data = [r for r in rows[2:] if len(r) > iexe and r[ia].startswith("0x")]
base = min(int(r[ia], 16) for r in data)
tot = sum(int(r[isamp] or 0) for r in data)
order = sorted(range(len(data)), key=lambda i: -int(data[i][isamp] or 0))[:top]
for i in order:
    r = data[i]
    s = int(r[isamp] or 0)
    why = sorted(((int(r[j] or 0), hdr[j][6:]) for j in reasons), reverse=True)[:2]
    print(f"{s / tot * 100:5.2f}% {hex(int(r[ia], 16) - base):>8} exe={int(r[iexe] or 0):9d} {r[isrc][:58]:58s} "
          + " ".join(f"{w}:{n}" for n, w in why if n))
    for k in range(max(0, i - ctx), i):
        print(f"{'':16s}{hex(int(data[k][ia], 16) - base):>8} {data[k][isrc][:70]}")
