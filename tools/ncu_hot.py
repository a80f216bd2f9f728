"""Summarise an `ncu --page source --csv --print-source sass` export: top SASS lines by a stall column.
usage: python tools/ncu_hot.py file.csv [stall_col] [n]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
col = sys.argv[2] if len(sys.argv) > 2 else "stall_long_sb"
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
hdr = rows[1]
ia, isrc, ic = hdr.index("Address"), hdr.index("Source"), hdr.index(col)
iall = hdr.index("Warp Stall Sampling (All Samples)")
body = [r for r in rows[2:] if len(r) == len(hdr) and r[0].startswith('0x')]
tot = sum(float(r[iall] or 0) for r in body)
tc = sum(float(r[ic] or 0) for r in body)
print(f"total samples {tot:.0f}; {col} {tc:.0f} ({100 * tc / max(tot, 1):.1f}%)")
for i, r in sorted(enumerate(body), key=lambda x: -float(x[1][ic] or 0))[:n]:
    ctx = " | ".join(b[isrc].strip()[:38] for b in body[max(0, i - 2):i])
    print(f"{float(r[ic] or 0):7.0f}  {i:5d} {r[isrc].strip()[:60]:60s}  <- {ctx}")
