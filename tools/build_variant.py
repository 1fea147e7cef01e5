"""Dev tool: build libprg with extra -D flags into build/<name>.so (A/B via PRG_LIB).
usage: python tools/build_variant.py NAME -DFOO=1 [-DBAR=2 ...]"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1603_01876_b200.build as B  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
objdir = os.path.join(B.ROOT, "build", "var_" + name)
os.makedirs(objdir, exist_ok=True)
objs = []
jobs = []
for src in B.CU_SOURCES:
    o = os.path.join(objdir, src.replace(".cu", ".o"))
    objs.append(o)
    jobs.append([B.NVCC] + B.NVCC_FLAGS + defs + ["-c", os.path.join(B.CSRC, src), "-o", o])
from concurrent.futures import ThreadPoolExecutor  # noqa: E402

with ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
    list(ex.map(B._run, jobs))
out = os.path.join(B.ROOT, "build", name + ".so")
B._run([B.NVCC] + B.ARCH + ["-shared", "-o", out] + objs + ["-lcudart"])
print(out)
