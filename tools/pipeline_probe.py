import sys, time, json, tempfile
sys.path.insert(0, "paper_1603_01876_b200/python"); sys.path.insert(0, ".")
import prpipe
for S in (16, 20):
    with tempfile.TemporaryDirectory() as d:
        t = time.time()
        rep = prpipe.run_pipeline(scale=S, seed=1, data_dir=d + "/data")
        print(S, round(time.time() - t, 2), json.dumps([(k["name"], round(k["elapsed_seconds"], 4), "%.3g" % k["rate_edges_per_sec"]) for k in rep["kernels"]]))
