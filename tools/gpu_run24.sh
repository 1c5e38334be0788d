timeout 900 python -m pytest tests/test_parity.py -x -q -k "pipelined or graph" 2>&1 | tail -5 > gpurun_out/r24_pytest.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r24_bench.json 2> gpurun_out/r24_bench.err
timeout 900 python bench.py --config c2 --no-cpu-baseline > gpurun_out/r24_bench2.json 2>> gpurun_out/r24_bench.err
