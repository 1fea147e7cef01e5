# quick GPU check (dev tool): a pytest selection, then A/B bench specs
#   bash tools/gpu_quick.sh "<pytest -k expr>" "name:ENV=.." ...
set -x
K="$1"; shift
if [ -n "$K" ]; then timeout 900 python -m pytest tests -x -q -m gpu -k "$K" > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_quick.log; fi
bash tools/ab_env.sh "$@"
