# full GPU suite + timings of every config + count mode (after a default change)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/k_build.log 2>&1
timeout 1800 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -6 > gpurun_out/k_pytest.log
for c in c3 c5 c2 c4 c1; do timeout 300 python tools/ab_flags.py $c 9 0 >> gpurun_out/k_time.log 2>&1; done
timeout 600 python bench.py --config c3 --mode count --steps 10 --warmup 3 > gpurun_out/k_count.json 2> gpurun_out/k_count.err
