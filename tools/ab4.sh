# bash tools/ab4.sh "A:" "B:PRG_NCTR=8" ...  (SpMV over pool placements)
for spec in "$@"; do
  v=${spec%%:*}; envs=${spec#*:}
  env $envs TAG="$spec" PRG_LIB=build/ab/libprg_$v.so python tools/exp_spmv4.py
done
