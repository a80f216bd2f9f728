"""Per-source-line stall summary of one kernel in an ncu report (--import-source on, -lineinfo):
    python tools/ncu_lines.py <report.ncu-rep> [top N]
Reads `ncu -i --page source --csv --print-source cuda,sass` and prints the CUDA lines with the
most warp-stall samples and their top stall reasons."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
lines, hdr, fname = [], None, "?"
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].rsplit("/", 1)[-1]
    elif r[0] == "Line No":
        hdr = r
    elif hdr and r[0].isdigit():
        # ncu does not escape quotes inside source text: index the metrics from the right
        lines.append((fname, [r[0], ",".join(r[1:len(r) - len(hdr) + 2])] + r[len(r) - len(hdr) + 2:]))
i_s = hdr.index("Warp Stall Sampling (All Samples)")
i_x = hdr.index("Instructions Executed")
stall_cols = [i for i, c in enumerate(hdr) if c.startswith("stall_") and "Not Issued" not in c]
tot = sum(float(r[i_s] or 0) for _, r in lines if r[i_s] not in ('-', ''))
print(f"total stall samples {tot:.0f}")
num = lambda v: float(v) if v not in ("-", "") else 0.0
lines = [(f, r) for f, r in lines if num(r[i_s]) > 0]
for f, r in sorted(lines, key=lambda fr: -num(fr[1][i_s]))[:top]:
    s = float(r[i_s] or 0)
    st = sorted(((hdr[i][6:], num(r[i])) for i in stall_cols), key=lambda kv: -kv[1])[:3]
    print(f"{f}:{r[0]:>5} {100 * s / tot:5.1f}%  inst {r[i_x]:>10}  {' '.join(f'{k}={100 * v / max(s, 1):.0f}%' for k, v in st)}"
          f"  | {r[1].strip()[:80]}")
