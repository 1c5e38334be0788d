# fused count+emit A/B: tree (fused vs DDM_EMIT_UNFUSED) and timing-only variants; args: configs
for c in "$@"; do
  echo "== tree $c" >> gpurun_out/fab.log
  timeout 300 python tools/ab_flags.py $c 7 0 0x800 >> gpurun_out/fab.log 2>&1
  timeout 300 python tools/time_config.py $c 3 2>&1 | sed -n 3,8p >> gpurun_out/fab.log
  for v in nolb noemit minb2; do
    echo "== $v $c" >> gpurun_out/fab.log
    DDM_LIB=$PWD/variants/libddm_$v.so timeout 300 python tools/time_config.py $c 3 2>&1 | sed -n 3,8p >> gpurun_out/fab.log
  done
done
timeout 900 python -m pytest tests/test_parity.py -x -q -k "fused or walk_capacity or graph" 2>&1 | tail -3 >> gpurun_out/fab.log
