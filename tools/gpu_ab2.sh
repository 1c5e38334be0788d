# full GPU suite + A/B timing of the tree against variants/libddm_<name>.so; args: "cfgs" names...
cfgs=$1; shift
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab2_build.log 2>&1
timeout 1500 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -8 > gpurun_out/ab2_pytest.log
for c in $cfgs; do
  echo "== tree $c" >> gpurun_out/ab2.log
  timeout 300 python tools/ab_flags.py $c 9 0 >> gpurun_out/ab2.log 2>&1
  timeout 300 python tools/time_config.py $c 3 2>&1 | sed -n 3,9p >> gpurun_out/ab2.log
  for v in "$@"; do
    echo "== $v $c" >> gpurun_out/ab2.log
    DDM_LIB=$PWD/variants/libddm_$v.so timeout 300 python tools/ab_flags.py $c 9 0 >> gpurun_out/ab2.log 2>&1
    DDM_LIB=$PWD/variants/libddm_$v.so timeout 300 python tools/time_config.py $c 3 2>&1 | sed -n 3,9p >> gpurun_out/ab2.log
  done
done
