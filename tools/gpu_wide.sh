# LsWide A/B (env DDM_LS_WIDE_SPANS=0 disables it) + parity subset
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/w_build.log 2>&1
timeout 1500 python -m pytest tests/test_parity.py -x -q -k "msd or c1_full or c2_full or tie or fuzz or small or ragged or long or chunk or events or index or validation or capacity" 2>&1 | tail -5 > gpurun_out/w_pytest.log
for c in c1 c2 c4; do
  for e in 0 296; do
    echo "== wide_spans=$e $c" >> gpurun_out/w.log
    DDM_LS_WIDE_SPANS=$e timeout 300 python tools/ab_flags.py $c 15 0 >> gpurun_out/w.log 2>&1
    DDM_LS_WIDE_SPANS=$e timeout 300 python tools/time_config.py $c 5 2>&1 | sed -n 3,8p >> gpurun_out/w.log
  done
done
