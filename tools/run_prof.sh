set -x
python bench.py > gpurun_out/bench_r01.json 2> gpurun_out/bench_r01.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01.csv python bench.py --steps 1 --warmup 1 --e2e-steps 1 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:spmv_sell -s 5 -c 1 -o gpurun_out/prof_spmv_r01 python bench.py --steps 1 --warmup 1 --e2e-steps 1 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
ncu --set full --clock-control none -k regex:local_sort -s 0 -c 1 -o gpurun_out/prof_local_r01 python bench.py --steps 1 --warmup 0 --e2e-steps 1 --no-cpu-baseline > gpurun_out/ncu_full2.log 2>&1
ncu --set full --clock-control none -k regex:k2_pass_b -s 0 -c 1 -o gpurun_out/prof_k2b_r01 python bench.py --steps 1 --warmup 0 --e2e-steps 1 --no-cpu-baseline > gpurun_out/ncu_full3.log 2>&1
tail -c 400 gpurun_out/bench_r01.json
