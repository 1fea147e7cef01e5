# Round artifacts, part A (dev tool): GPU suite + smoke + bench lines + launch list (small outputs).
set -x
TAG=${1:-r02}
export PRG_PARITY_LOG=gpurun_out/${TAG}_drift.jsonl
rm -f $PRG_PARITY_LOG
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/${TAG}_bench_s24.log 2>&1; echo "bench rc=$?"
timeout 900 python bench.py --scale 26 --steps 3 --warmup 3 --no-cpu-baseline --no-pipeline-io --e2e-steps 1 > gpurun_out/${TAG}_bench_s26.log 2>&1; echo "bench26 rc=$?"
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-pipeline-io --e2e-steps 1"
$B > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/${TAG}_launches_s24.csv $B > gpurun_out/${TAG}_ncu_l.log 2>&1
echo "launches rc=$?"
