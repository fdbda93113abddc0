"""Copy one measurement pass (tools/measure_round.sh TAG) from gpurun_out/ into profiles/ (dev tool):
ncu --set full summaries of the two step kernels, the launch list of the bench command, per-launch DRAM traffic
(profiles/traffic.json, read by bench.py for roofline.traffic), the bench line and the GPU pytest log.

    python tools/post_round.py r01d [--fg 16] [--shot-batch 16]
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
ap.add_argument("--fg", type=int, default=16)
ap.add_argument("--shot-batch", type=int, default=16)
a = ap.parse_args()
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")
UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}

traffic = {"source": f"ncu --set full, {a.tag} (profiles/{a.tag}_ncu_*.txt), cfg1 S={a.shot_batch} FG={a.fg} BWD_FG=2"}
for kern, short in (("fwd_step_kernel", "fwd"), ("bwd_step_kernel", "bwd")):
    rep = os.path.join(G, f"prof_{short}_{a.tag}.ncu-rep")
    res = summarise(rep)
    with open(os.path.join(P, f"{a.tag}_ncu_{short}_step.txt"), "w") as f:
        for d in res:
            f.write(f"--- {d['kernel']}\n")
            for k in KEYS:
                if k in d:
                    f.write(f"  {k:80s} {d[k]} {d[k + '@unit']}\n")
    b = [d["dram__bytes_read.sum"] * UNIT[d["dram__bytes_read.sum@unit"]] +
         d["dram__bytes_write.sum"] * UNIT[d["dram__bytes_write.sum@unit"]] for d in res]
    t = [d["gpu__time_duration.sum"] for d in res]
    traffic[kern] = {"config": {"workload": "cfg1", "shot_batch": a.shot_batch, "field_group": a.fg},
                     "dram_bytes_per_launch": sum(b) / len(b), "duration_us_ncu": sum(t) / len(t)}
json.dump(traffic, open(os.path.join(P, "traffic.json"), "w"), indent=1)

rows = [r for r in csv.reader(open(os.path.join(G, f"launches_{a.tag}.csv"))) if len(r) > 5]
hdr = rows[0]
i_name, i_val = hdr.index("Kernel Name"), hdr.index("Metric Value")
per = collections.defaultdict(list)
for r in rows[1:]:
    per[r[i_name].split("(")[0]].append(float(r[i_val].replace(",", "")) / 1000.0)
tot = sum(sum(v) for v in per.values())
with open(os.path.join(P, f"{a.tag}_launches.csv"), "w") as f:
    f.write(f"# ncu launch list (gpu__time_duration.sum, --clock-control none, cold-cache serialised), {a.tag}\n"
            "# command: python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e ; ncu -s 12000 -c 4200\n"
            "kernel,launches,mean_us,share_of_listed_time\n")
    for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
        f.write(f"{k},{len(v)},{sum(v) / len(v):.2f},{sum(v) / tot:.4f}\n")
for src, dst in ((f"bench_{a.tag}.json", f"{a.tag}_bench.json"), (f"pytest_gpu_{a.tag}.log", f"{a.tag}_pytest_gpu.log")):
    if os.path.exists(os.path.join(G, src)):
        shutil.copy(os.path.join(G, src), os.path.join(P, dst))
print(json.dumps(traffic, indent=1))
print(open(os.path.join(P, f"{a.tag}_launches.csv")).read())
