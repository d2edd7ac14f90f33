"""Per-source-line stall samples / executed instructions from an ncu report (cuda,sass view).

  python tools/ncu_lines.py report.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
res = []
cur_file = None
hdr = None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr) or r[0] == "" or r[0] == "Function Name":
        continue
    try:
        smp = float(r[4] or 0)
        ex = float(r[7] or 0)
    except ValueError:
        continue
    res.append((smp, ex, f"{cur_file}:{r[0]}", r[1].strip()[:100]))
tot = sum(x[0] for x in res)
totx = sum(x[1] for x in res)
print(f"total samples {tot:.0f}  warp instructions {totx:.0f}")
for smp, ex, loc, src in sorted(res, reverse=True)[:top]:
    print(f"{smp:7.0f} {100 * smp / max(tot, 1):5.1f}% {ex:11.0f} {100 * ex / max(totx, 1):5.1f}%  {loc:22s} {src}")
