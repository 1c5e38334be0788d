# full GPU test suite + smoke + default bench
timeout 1800 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -4 > gpurun_out/c_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/c_bench.json 2> gpurun_out/c_bench.err
