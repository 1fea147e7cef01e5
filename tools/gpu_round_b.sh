# Round artifacts, part B (dev tool): full ncu captures (each after the same command ran plainly).
# Summaries are written on the box (the reports themselves exceed what gpurun copies back).
set -x
TAG=${1:-r02}
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-pipeline-io --e2e-steps 1"
$B > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:spmv_sell -s 30 -c 1 -o /tmp/${TAG}_spmv_s24 -f $B > gpurun_out/${TAG}_ncu_s.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"local_s|k2_pass|sell_fill|gather_y|l1_scatter|key_build|seg_scatter" -c 24 -o /tmp/${TAG}_kernels_s24 -f $B > gpurun_out/${TAG}_ncu_k.log 2>&1
echo "ncu rc=$?"
B26="python bench.py --scale 26 --steps 1 --warmup 1 --no-cpu-baseline --no-pipeline-io --e2e-steps 1"
$B26 > gpurun_out/${TAG}_plain26.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:spmv_sell -s 30 -c 1 -o /tmp/${TAG}_spmv_s26 -f $B26 > gpurun_out/${TAG}_ncu_s26.log 2>&1
echo "ncu26 rc=$?"
python tools/ncu_summary.py /tmp/${TAG}_spmv_s24.ncu-rep 15 > gpurun_out/${TAG}_ncu_spmv_s24.txt 2>&1
python tools/ncu_summary.py /tmp/${TAG}_spmv_s26.ncu-rep 15 > gpurun_out/${TAG}_ncu_spmv_s26.txt 2>&1
python tools/ncu_summary.py /tmp/${TAG}_kernels_s24.ncu-rep 8 > gpurun_out/${TAG}_ncu_kernels_s24.txt 2>&1
cp profiles/ncu_traffic.json /tmp/ncu_traffic_before.json
python tools/ncu_traffic.py /tmp/${TAG}_spmv_s24.ncu-rep --scale 24 --summary ${TAG}_ncu_spmv_s24.txt
python tools/ncu_traffic.py /tmp/${TAG}_spmv_s26.ncu-rep --scale 26 --summary ${TAG}_ncu_spmv_s26.txt
cp profiles/ncu_traffic.json gpurun_out/ncu_traffic.json
cp /tmp/${TAG}_spmv_s24.ncu-rep gpurun_out/ 2>/dev/null
ls -la /tmp/*.ncu-rep
