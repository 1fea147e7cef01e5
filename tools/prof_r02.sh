# Round-2 ncu captures (dev tool; under gpurun). Every ncu command follows the
# same command run plainly (exit 0) first, as the profiling recipe requires.
set -x
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-pipeline-io --e2e-steps 1"
$B > gpurun_out/r02_plain_s24.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r02_launches_s24.csv $B > gpurun_out/ncu_l.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:spmv_sell -s 30 -c 1 -o gpurun_out/r02_spmv_s24 -f $B > gpurun_out/ncu_s24.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"local_sort|k2_pass|sell_fill|gather_y|l1_scatter|key_build" -c 16 -o gpurun_out/r02_kernels_s24 -f $B > gpurun_out/ncu_k24.log 2>&1
echo "s24 rc=$?"
B26="python bench.py --scale 26 --steps 1 --warmup 1 --no-cpu-baseline --no-pipeline-io --e2e-steps 1"
$B26 > gpurun_out/r02_plain_s26.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:spmv_sell -s 30 -c 1 -o gpurun_out/r02_spmv_s26 -f $B26 > gpurun_out/ncu_s26.log 2>&1
echo "s26 rc=$?"
ls -la gpurun_out/*.ncu-rep gpurun_out/*.csv
