# Round artifacts on one GPU box in ONE call (dev tool) — superseded by gpu_round_a.sh + gpu_round_b.sh: the
# reports this writes under gpurun_out/ now exceed the 64 MiB gpurun copies back.
# Every ncu command runs after the same command exited 0 without ncu.
set -x
TAG=${1:-r02}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
export PRG_PARITY_LOG=gpurun_out/${TAG}_drift.jsonl
rm -f $PRG_PARITY_LOG
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/${TAG}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/${TAG}_bench_s24.log 2>&1; echo "bench rc=$?"
timeout 900 python bench.py --scale 26 --steps 3 --warmup 3 --no-cpu-baseline --no-pipeline-io --e2e-steps 1 > gpurun_out/${TAG}_bench_s26.log 2>&1; echo "bench26 rc=$?"
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-pipeline-io --e2e-steps 1"
$B > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/${TAG}_launches_s24.csv $B > gpurun_out/${TAG}_ncu_l.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:spmv_sell -s 30 -c 1 -o gpurun_out/${TAG}_spmv_s24 -f $B > gpurun_out/${TAG}_ncu_s.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"local_sort|k2_pass|sell_fill|gather_y|l1_scatter|key_build|seg_scatter" -c 20 -o gpurun_out/${TAG}_kernels_s24 -f $B > gpurun_out/${TAG}_ncu_k.log 2>&1
echo "ncu rc=$?"
B26="python bench.py --scale 26 --steps 1 --warmup 1 --no-cpu-baseline --no-pipeline-io --e2e-steps 1"
$B26 > gpurun_out/${TAG}_plain26.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:spmv_sell -s 30 -c 1 -o gpurun_out/${TAG}_spmv_s26 -f $B26 > gpurun_out/${TAG}_ncu_s26.log 2>&1
echo "ncu26 rc=$?"
