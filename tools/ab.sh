# A/B timing between library builds / env settings (dev tool): bash tools/ab.sh "A:" "B:PRG_X=1" ...
for spec in "$@"; do
  v=${spec%%:*}; envs=${spec#*:}
  env $envs PRG_LIB=build/ab/libprg_$v.so python bench.py --no-cpu-baseline --e2e-steps 1 > gpurun_out/ab.log 2>&1
  python -c "
import json;d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]);k=d['kernel_ms'];st=d['stage_ms']
print('$spec','k1 %.3f k2f %.3f k2c %.3f k3 %.3f cold %.3f'%(st['k1_sort'],st['k2_filter_csr'],st['k2_csc_build'],st['k3_pagerank'],d['k3_cold']['ms']),{x:round(k[x]['avg_ms'],4) for x in k if x in ('k3_spmv','k3_permute','k2_pass_a','k2_pass_b')})"
done
