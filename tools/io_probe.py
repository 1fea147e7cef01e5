"""Dev tool: phase times of the drop-in's I/O-inclusive run_pipeline records (PRG_IO_DEBUG=1)."""
import os, sys, tempfile, time
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_1603_01876_b200", "python"))
import prpipe
S = int(sys.argv[1]) if len(sys.argv) > 1 else 20
with tempfile.TemporaryDirectory() as d:
    prpipe.run_pipeline(scale=10, seed=1, data_dir=os.path.join(d, "warm"))
    for rep in range(2):
        r = prpipe.run_pipeline(scale=S, seed=1, data_dir=os.path.join(d, f"data{rep}"))
        print({k["name"]: round(k["elapsed_seconds"], 4) for k in r["kernels"]}, flush=True)
