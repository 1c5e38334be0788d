# time c3 (profiled breakdown + official A/B) for the in-tree build and each variants/libddm_<name>.so
# usage: gpu_variants.sh cfg name...
cfg=$1; shift
echo "== tree" > gpurun_out/v.log
timeout 300 python tools/time_config.py $cfg 5 2>&1 | head -12 >> gpurun_out/v.log
timeout 300 python tools/ab_flags.py $cfg 7 0 >> gpurun_out/v.log 2>&1
for v in "$@"; do
  echo "== $v" >> gpurun_out/v.log
  DDM_LIB=$PWD/variants/libddm_$v.so timeout 300 python tools/time_config.py $cfg 5 2>&1 | head -12 >> gpurun_out/v.log
  DDM_LIB=$PWD/variants/libddm_$v.so timeout 300 python tools/ab_flags.py $cfg 7 0 >> gpurun_out/v.log 2>&1
done
