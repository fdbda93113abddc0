"""Per-source-line instruction counts and stall samples from an ncu report (dev tool):
python tools/src_lines.py report.ncu-rep [kernel-regex] [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]
if len(sys.argv) > 2 and sys.argv[2]:
    cmd += ["-k", "regex:" + sys.argv[2]]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(cmd, capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname = None
res = []
hdr = None
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    elif r and r[0] == "Line No":
        hdr = r
    elif hdr and r and r[0] and r[0].isdigit() and len(r) == len(hdr):
        n = int(r[hdr.index("Instructions Executed")] or 0)
        s = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        if n or s:
            res.append((n, s, f"{fname}:{r[0]}", r[1].strip()[:90]))
tot = sum(x[0] for x in res)
ts = sum(x[1] for x in res)
print(f"total {tot} inst, {ts} samples")
for n, s, loc, src in sorted(res, reverse=True)[:top]:
    print(f"{100.0*n/tot:5.1f}% {100.0*s/max(ts,1):5.1f}%s  {loc:22s} {src}")
