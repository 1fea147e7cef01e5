# compute-sanitizer over the whole device path; logs in gpurun_out/
set -x
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 900 $CS --tool memcheck --error-exitcode 9 python tools/sanitize_driver.py 12 > gpurun_out/sanitize_memcheck.log 2>&1; echo "memcheck rc=$?"
timeout 1500 $CS --tool racecheck --racecheck-report all --error-exitcode 9 python tools/sanitize_driver.py 10 > gpurun_out/sanitize_racecheck.log 2>&1; echo "racecheck rc=$?"
timeout 900 $CS --tool synccheck --error-exitcode 9 python tools/sanitize_driver.py 12 > gpurun_out/sanitize_synccheck.log 2>&1; echo "synccheck rc=$?"
timeout 900 $CS --tool initcheck --error-exitcode 9 python tools/sanitize_driver.py 10 > gpurun_out/sanitize_initcheck.log 2>&1; echo "initcheck rc=$?"
tail -3 gpurun_out/sanitize_*.log
