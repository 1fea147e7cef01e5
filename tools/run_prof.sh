# Round profiling pass (run on the GPU box via gpurun from the repo root).
# Each ncu command runs only after the same bench command exited 0 without ncu.
set -x
R=${1:-r01}
python bench.py > gpurun_out/bench_$R.json 2> gpurun_out/bench_$R.err || exit 1
python bench.py --steps 1 --warmup 1 --e2e-steps 1 --no-cpu-baseline > gpurun_out/bench_short.json 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$R.csv \
    python bench.py --steps 1 --warmup 1 --e2e-steps 1 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:spmv_sell -s 25 -c 1 \
    -o gpurun_out/prof_spmv_$R python bench.py --steps 1 --warmup 1 --e2e-steps 1 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"local_sort|l1_scatter|seg_scatter|k2_pass|key_build|row_base|sell_fill" -s 0 -c 14 \
    -o gpurun_out/prof_prep_$R python bench.py --steps 1 --warmup 0 --e2e-steps 1 --no-cpu-baseline > gpurun_out/ncu_full2.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k regex:"CscDst|key_build|sell_fill" -c 3 -o gpurun_out/prof_k3prep_$R python tools/prof_driver.py k3 24 \
    > gpurun_out/ncu_full3.log 2>&1
tail -c 600 gpurun_out/bench_$R.json
