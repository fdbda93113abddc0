"""Copy one measurement pass (tools/measure_round.sh TAG) from gpurun_out/ into profiles/ (dev tool):
ncu --set full summaries of the two step kernels at the bench's launch configuration, per-launch DRAM traffic
(profiles/traffic.json records, read by bench.py for roofline.traffic / dram_frac), the launch list of the bench
command, the bench / evidence lines and the GPU pytest log.

    python tools/post_round.py r02 [--workload cfg3 --shot-batch 16 --K 32]
"""
import argparse
import collections
import csv
import json
import os
import shutil
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, HERE)
from ncu_summary import KEYS, summarise  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("tag")
ap.add_argument("--workload", default="cfg3")
ap.add_argument("--shot-batch", type=int, default=16)
ap.add_argument("--K", type=int, default=32)
a = ap.parse_args()
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")
UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}

tpath = os.path.join(P, "traffic.json")
try:
    traffic = json.load(open(tpath))
    if "records" not in traffic:
        traffic = {"records": []}
except Exception:
    traffic = {"records": []}
CAPTURES = [  # (report stem, summary name, workload, shot batch, K, command)
    ("fwd", "fwd", a.workload, a.shot_batch, a.K, "tools/profile_step.py --config 3 --shots 16 --nt 40"),
    ("bwd", "bwd", a.workload, a.shot_batch, a.K, "tools/profile_step.py --config 3 --shots 16 --nt 40"),
    ("fwd_cfg4", "cfg4grid_fwd", "cfg4", 4, 64,
     "tools/profile_step.py --config 4 --shots 4 --nt 12"),
    ("bwd_cfg4", "cfg4grid_bwd", "cfg4", 4, 64,
     "tools/profile_step.py --config 4 --shots 4 --nt 12"),
]
for stem, short, workload, sb, K, cmd in CAPTURES:
    rep = os.path.join(G, f"prof_{stem}_{a.tag}.ncu-rep")
    if not os.path.exists(rep):
        continue
    res = summarise(rep)
    with open(os.path.join(P, f"{a.tag}_ncu_{short}.txt"), "w") as f:
        f.write(f"# ncu --set full --clock-control none, {workload} S={sb} K={K} ({cmd}), {a.tag}\n")
        for d in res:
            f.write(f"--- {d['kernel']}\n")
            for k in KEYS:
                if k in d:
                    f.write(f"  {k:80s} {d[k]} {d[k + '@unit']}\n")
    for d in res:
        b = (d["dram__bytes_read.sum"] * UNIT[d["dram__bytes_read.sum@unit"]] +
             d["dram__bytes_write.sum"] * UNIT[d["dram__bytes_write.sum@unit"]])
        t = d["gpu__time_duration.sum"] * {"ns": 1e-3, "us": 1.0, "ms": 1e3}.get(d["gpu__time_duration.sum@unit"], 1.0)
        rec = {"kernel": d["kernel"].replace("hvk::", ""), "workload": workload, "shot_batch": sb,
               "K": K, "dram_bytes_per_launch": b, "duration_us_ncu": t,
               "source": f"ncu --set full, {a.tag} (profiles/{a.tag}_ncu_{short}.txt)"}
        traffic["records"] = [r for r in traffic["records"]
                              if not (r["kernel"] == rec["kernel"] and r["workload"] == rec["workload"]
                                      and r["shot_batch"] == rec["shot_batch"] and r["K"] == rec["K"])]
        traffic["records"].append(rec)
json.dump(traffic, open(tpath, "w"), indent=1)

lpath = os.path.join(G, f"launches_{a.tag}.csv")
if os.path.exists(lpath):
    rows = [r for r in csv.reader(open(lpath)) if len(r) > 5]
    hdr = rows[0]
    i_name, i_val = hdr.index("Kernel Name"), hdr.index("Metric Value")
    per = collections.defaultdict(list)
    for r in rows[1:]:
        per[r[i_name].split("(")[0].replace("hvk::", "")].append(float(r[i_val].replace(",", "")) / 1000.0)
    tot = sum(sum(v) for v in per.values())
    with open(os.path.join(P, f"{a.tag}_launches.csv"), "w") as f:
        f.write(f"# ncu launch list (gpu__time_duration.sum, --clock-control none, cold-cache serialised), {a.tag}\n"
                "# command: python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e ; ncu -s 2000 -c 6000\n"
                "kernel,launches,mean_us,share_of_listed_time\n")
        for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
            f.write(f"{k},{len(v)},{sum(v) / len(v):.2f},{sum(v) / tot:.4f}\n")
    print(open(os.path.join(P, f"{a.tag}_launches.csv")).read())
for src in os.listdir(G):
    if src.endswith(f"_{a.tag}.json") or src == f"pytest_gpu_{a.tag}.log" or src == f"smoke_{a.tag}.log":
        shutil.copy(os.path.join(G, src), os.path.join(P, f"{a.tag}_{src.replace('_' + a.tag, '')}"))
print(json.dumps(traffic, indent=1))
