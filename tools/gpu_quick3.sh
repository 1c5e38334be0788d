# quick GPU check of a change: build, a parity subset (-k EXPR), timings of the given configs
k=${1:-"fused or walk or c3_full or c5 or long or stab_walk or capacity or ragged or c2_full or fuzz or c1"}
shift
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/q3_build.log 2>&1
timeout 1200 python -m pytest tests/test_parity.py -x -q -k "$k" 2>&1 | tail -15 > gpurun_out/q3_pytest.log
for c in "$@"; do timeout 600 python tools/time_config.py $c 5 > gpurun_out/q3_time_$c.log 2>&1; done
