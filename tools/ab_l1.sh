# sort level-1 A/B (dev tool)
for spec in "$@"; do
  v=${spec%%:*}; envs=${spec#*:}
  env $envs PRG_LIB=build/ab/libprg_$v.so python bench.py --no-cpu-baseline --no-pipeline-io --e2e-steps 1 > gpurun_out/ab.log 2>&1
  python -c "
import json;d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]);k=d['kernel_ms'];st=d['stage_ms']
print('$spec','k1 %.3f k2c %.3f'%(st['k1_sort'],st['k2_csc_build']),{x:round(v['avg_ms'],3) for x,v in k.items() if 'l1_' in x})"
done
