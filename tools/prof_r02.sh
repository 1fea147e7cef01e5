# Round-2 ncu captures (dev tool). Run under gpurun; reports land in gpurun_out/.
set -x
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-pipeline-io --e2e-steps 1"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"local_sort|k2_pass|sell_fill|l1_scatter|seg_scatter|l1_hist|seg_hist" -s 0 -c 16 -o gpurun_out/r02_prep -f $B > gpurun_out/ncu_prep.log 2>&1
echo "ncu rc=$?"
ls -la gpurun_out
