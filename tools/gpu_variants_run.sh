# usage: bash tools/gpu_variants_run.sh TAG CFG REPS lib1 lib2 ... (run on the GPU box)
tag=$1; cfg=$2; reps=$3; shift 3
for lib in default "$@"; do
  if [ "$lib" = default ]; then unset DDM_LIB; else export DDM_LIB=$PWD/variants/libddm_$lib.so; fi
  timeout 600 python tools/variant_time.py $cfg $reps >> gpurun_out/${tag}_$cfg.jsonl 2>> gpurun_out/${tag}_$cfg.err
done
unset DDM_LIB
