for spec in "0:16384" "2:16384" "3:16384" "4:16384" "5:16384" "2:4096" "2:65536" "4:65536" "3:65536"; do
 v=${spec%%:*}; h=${spec#*:}
 TAG="variant=$v hot=$h" PRG_SPMV_VARIANT=$v PRG_HOT_ROWS=$h timeout 300 python tools/exp_spmv4.py 2>&1 | tail -1
done
