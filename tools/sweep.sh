# dev: env sweep of the bench (K3 stage times); usage: bash tools/sweep.sh VAR v1 v2 ...
var=$1; shift
for v in "$@"; do
  env $var=$v timeout 300 python bench.py --no-cpu-baseline --e2e-steps 1 > gpurun_out/sw.log 2>&1
  tail -1 gpurun_out/sw.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernel_ms']; print('$var=$v', round(d['stage_ms']['k3_pagerank'],3), {x:round(k[x]['avg_ms'],3) for x in ('k3_spmv','k3_prep_sell','k3_prep')})"
done
