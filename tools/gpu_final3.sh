# round-end evidence in one call: A/B timing of the tree against variants (optional),
# full GPU suite + smoke + tools/gpu_evidence.sh TAG, then the ncu reports turned into
# text ON THE BOX (gpurun_out/ comes back only under 64 MiB; the .ncu-rep files are deleted)
# usage: bash tools/gpu_final3.sh TAG "cfgs" variants...
tag=$1; cfgs=$2; shift 2
o=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $o/${tag}_build0.log 2>&1
for c in $cfgs; do
  echo "== tree $c" >> $o/${tag}_ab.log
  timeout 300 python tools/ab_flags.py $c 9 0 >> $o/${tag}_ab.log 2>&1
  timeout 300 python tools/time_config.py $c 3 2>&1 | sed -n 3,12p >> $o/${tag}_ab.log
  for v in "$@"; do
    echo "== $v $c" >> $o/${tag}_ab.log
    DDM_LIB=$PWD/variants/libddm_$v.so timeout 300 python tools/ab_flags.py $c 9 0 >> $o/${tag}_ab.log 2>&1
    DDM_LIB=$PWD/variants/libddm_$v.so timeout 300 python tools/time_config.py $c 3 2>&1 | sed -n 3,12p >> $o/${tag}_ab.log
  done
done
timeout 1800 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -6 > $o/${tag}_gpu_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > $o/${tag}_smoke.log 2>&1
bash tools/gpu_evidence.sh $tag
mkdir -p $o/${tag}_prof
for k in msd_pass local_sort count emit dd_stage; do
  [ -f $o/${tag}_$k.ncu-rep ] || continue
  ncu -i $o/${tag}_$k.ncu-rep --page details > $o/${tag}_prof/${k}_ncu_full.txt 2>/dev/null
  python tools/ncu_lines.py $o/${tag}_$k.ncu-rep "" 30 > $o/${tag}_prof/${k}_hot_lines.txt 2>/dev/null
  rm -f $o/${tag}_$k.ncu-rep
done
du -sh $o > $o/${tag}_du.txt
