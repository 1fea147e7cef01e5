"""Write profiles/ncu_traffic.json from an ncu --set full report of the SpMV
(dev tool): dram__bytes_read.sum + dram__bytes_write.sum of the captured launch.

usage: ncu_traffic.py REPORT --scale S [--tag k3_spmv] [--launch K]
Merges {scale: {tag: {...}}} into profiles/ncu_traffic.json (one capture per
kernel per scale; bench.py never reuses another scale's capture).
"""
import csv
import io
import json
import os
import subprocess
import sys

import argparse

ap = argparse.ArgumentParser()
ap.add_argument("report")
ap.add_argument("--scale", type=int, required=True)
ap.add_argument("--tag", default="k3_spmv")
ap.add_argument("--launch", type=int, default=0, help="row of the raw page (captured launch index)")
ap.add_argument("--summary", default=None, help="committed profiles/ summary of the same report (cited as the source)")
a = ap.parse_args()
rep = a.report
raw = list(csv.reader(io.StringIO(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"],
                                                 capture_output=True, text=True).stdout)))
h, units, v = raw[0], raw[1], raw[2 + a.launch]
d = dict(zip(h, v))
u = dict(zip(h, units))
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def get(k):
    return float(d[k].replace(",", "")) * scale.get(u[k], 1)


tot = get("dram__bytes_read.sum") + get("dram__bytes_write.sum")
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
path = os.path.join(root, "profiles", "ncu_traffic.json")
db = json.load(open(path)) if os.path.exists(path) else {}
db.setdefault(str(a.scale), {})[a.tag] = {"dram_bytes_per_launch": tot, "kernel": d.get("Kernel Name", ""),
                                          "source": a.summary or os.path.basename(rep), "report": os.path.basename(rep),
                                          "note": "one ncu --set full capture, cold-cache replay"}
with open(path, "w") as f:
    json.dump(db, f, indent=1, sort_keys=True)
print(json.dumps(db[str(a.scale)][a.tag]))
