# S=26 K3 A/B (dev tool): bash tools/ab26.sh "B:" "B:PRG_VCMAX=512" ...
for spec in "$@"; do
  v=${spec%%:*}; envs=${spec#*:}
  env $envs PRG_LIB=build/ab/libprg_$v.so python bench.py --scale 26 --steps 2 --warmup 1 --no-cpu-baseline --no-pipeline-io --e2e-steps 1 > gpurun_out/ab26.log 2>&1
  python -c "
import json;d=json.loads(open('gpurun_out/ab26.log').read().strip().splitlines()[-1]);k=d['kernel_ms'];st=d['stage_ms']
print('$spec','k1 %.2f k2f %.2f k2c %.2f k3 %.2f'%(st['k1_sort'],st['k2_filter_csr'],st['k2_csc_build'],st['k3_pagerank']),{x:round(k[x]['avg_ms'],4) for x in k if x in ('k3_spmv','k3_permute')})"
done
