set -x
B="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-pipeline-io --e2e-steps 0"
PRG_LOCAL_ALGO=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:local_sort -c 1 -o gpurun_out/r02_local_m64 -f $B > gpurun_out/ncu_local.log 2>&1
