# A/B timing of K3 between library builds / env settings (dev tool): bash tools/ab.sh "A:" "B:PRG_X=1" ...
for spec in "$@"; do
  v=${spec%%:*}; envs=${spec#*:}
  env $envs PRG_LIB=build/ab/libprg_$v.so python bench.py --no-cpu-baseline --e2e-steps 1 > gpurun_out/ab.log 2>&1
  python -c "
import json;d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]);k=d['kernel_ms'];print('$spec',round(d['stage_ms']['k3_pagerank'],3),round(d['k3_cold']['ms'],3),{x:round(k[x]['avg_ms'],4) for x in k if x in ('k3_spmv','k3_permute')}, d['clocks'])"
done
