"""Per-opcode instruction mix and stall samples from an ncu report's SASS source page (dev tool):
python tools/sass_mix.py report.ncu-rep [kernel-regex]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"]
if len(sys.argv) > 2:
    cmd += ["-k", "regex:" + sys.argv[2]]
out = subprocess.run(cmd, capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if r and r[0] == "Address")
i_src, i_ex, i_samp = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
ops = collections.Counter()
samp = collections.Counter()
tot = 0
for r in rows:
    if len(r) != len(hdr) or r[0] == "Address":
        continue
    src = r[i_src].strip()
    if src.startswith("@"):
        src = src.split(None, 1)[1]
    op = src.split()[0] if src else "?"
    n = int(r[i_ex] or 0)
    ops[op] += n
    samp[op] += int(r[i_samp] or 0)
    tot += n
ts = sum(samp.values())
print(f"total warp instructions {tot}, stall samples {ts}")
for op, n in ops.most_common(40):
    print(f"{op:28s} {n:12d} {100.0 * n / tot:6.2f}%   samples {100.0 * samp[op] / max(ts, 1):6.2f}%")
