timeout 1800 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -6 > gpurun_out/r23_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r23_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/r23_bench.json 2> gpurun_out/r23_bench.err
