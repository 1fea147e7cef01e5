set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
export PRG_PARITY_LOG=gpurun_out/drift_r02.jsonl
rm -f $PRG_PARITY_LOG
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench1.log 2>&1; echo "bench rc=$?"
tail -c 3000 gpurun_out/bench1.log
