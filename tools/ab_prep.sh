# CSC-build A/B (dev tool): bash tools/ab_prep.sh "B:" "B:PRG_X=1" ...
for spec in "$@"; do
  v=${spec%%:*}; envs=${spec#*:}
  env $envs PRG_LIB=build/ab/libprg_$v.so python bench.py --no-cpu-baseline --e2e-steps 1 > gpurun_out/ab.log 2>&1
  python -c "
import json;d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]);k=d['kernel_ms'];st=d['stage_ms']
print('$spec','k2c %.3f k3 %.3f'%(st['k2_csc_build'],st['k3_pagerank']),{x:round(v['avg_ms'],3) for x,v in k.items() if x.startswith('k3_prep') or x.startswith('k3t')})"
done
