# A/B timing of env-var knobs on one library build (dev tool):
#   bash tools/ab_env.sh "base:" "ldcs:PRG_K2_FLAGS=1" ...
for spec in "$@"; do
  v=${spec%%:*}; envs=${spec#*:}
  timeout 600 env $envs python bench.py --no-cpu-baseline --no-pipeline-io --e2e-steps 1 --steps 5 > gpurun_out/ab_$v.log 2>&1
  python - "$spec" "gpurun_out/ab_$v.log" <<'PY'
import json, sys
spec, path = sys.argv[1], sys.argv[2]
try:
    d = json.loads(open(path).read().strip().splitlines()[-1])
except Exception as e:
    print(spec, "FAILED", open(path).read()[-800:]); sys.exit()
k, st = d["kernel_ms"], d["stage_ms"]
keys = [x for x in k if x.startswith(("k1_", "k2_", "k3t_", "k3_prep", "k3_spmv", "k3_permute"))]
print(spec, "k1 %.3f k2f %.3f k2c %.3f k3 %.3f cold %.3f e2e %.1f ms" % (st["k1_sort"], st["k2_filter_csr"], st["k2_csc_build"],
      st["k3_pagerank"], d["k3_cold"]["ms"], d["e2e"]["seconds_per_step"] * 1e3))
print("   ", {x: round(k[x]["avg_ms"], 4) for x in sorted(keys)})
PY
done
