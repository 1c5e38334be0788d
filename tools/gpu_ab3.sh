# parity subset (-k EXPR) + A/B timing of the tree against variants; args: "k-expr" "cfgs" names...
k=$1; cfgs=$2; shift 2
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab3_build.log 2>&1
timeout 1500 python -m pytest tests/test_parity.py -x -q -k "$k" 2>&1 | tail -8 > gpurun_out/ab3_pytest.log
for c in $cfgs; do
  echo "== tree $c" >> gpurun_out/ab3.log
  timeout 300 python tools/ab_flags.py $c 9 0 >> gpurun_out/ab3.log 2>&1
  timeout 300 python tools/time_config.py $c 3 2>&1 | sed -n 3,9p >> gpurun_out/ab3.log
  for v in "$@"; do
    echo "== $v $c" >> gpurun_out/ab3.log
    DDM_LIB=$PWD/variants/libddm_$v.so timeout 300 python tools/ab_flags.py $c 9 0 >> gpurun_out/ab3.log 2>&1
    DDM_LIB=$PWD/variants/libddm_$v.so timeout 300 python tools/time_config.py $c 3 2>&1 | sed -n 3,9p >> gpurun_out/ab3.log
  done
done
