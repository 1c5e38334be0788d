timeout 1800 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -4 > gpurun_out/r17_pytest.log
for c in c3 c2 c4 c5; do timeout 1500 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/b_$c.json 2> gpurun_out/b_$c.err; done
