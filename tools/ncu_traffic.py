"""Write profiles/ncu_traffic.json from an ncu --set full report of the SpMV
(dev tool): dram__bytes_read.sum + dram__bytes_write.sum of the captured launch.

usage: ncu_traffic.py REPORT [--summary OUT.txt]
"""
import csv
import io
import json
import os
import subprocess
import sys

rep = sys.argv[1]
raw = list(csv.reader(io.StringIO(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"],
                                                 capture_output=True, text=True).stdout)))
h, units, v = raw[0], raw[1], raw[2]
d = dict(zip(h, v))
u = dict(zip(h, units))
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def get(k):
    return float(d[k].replace(",", "")) * scale.get(u[k], 1)


tot = get("dram__bytes_read.sum") + get("dram__bytes_write.sum")
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
out = {"k3_spmv": {"dram_bytes_per_launch": tot, "kernel": d.get("Kernel Name", ""),
                   "source": os.path.basename(rep), "note": "one ncu --set full capture, cold-cache replay"}}
with open(os.path.join(root, "profiles", "ncu_traffic.json"), "w") as f:
    json.dump(out, f, indent=1)
print(json.dumps(out))
