set -x
ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:spmv_sell -s 5 -c 1 -o gpurun_out/r01_spmv -f python tools/exp_spmv3.py > gpurun_out/ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gather_y -s 5 -c 1 -o gpurun_out/r01_gather -f python tools/exp_spmv3.py > gpurun_out/ncu2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k2_pass_b|k2_pass_a" -c 2 -o gpurun_out/r01_k2 -f python tools/exp_spmv3.py > gpurun_out/ncu3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:local_sort_kernel -c 1 -o gpurun_out/r01_k1local -f python tools/exp_spmv3.py > gpurun_out/ncu4.log 2>&1
ls -la gpurun_out
