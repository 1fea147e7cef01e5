set -x
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
tail -c 1500 gpurun_out/bench.log
bash tools/ab_env.sh "$@"
