timeout 1200 python -m pytest tests/test_parity.py -x -q -k "c5_full" 2>&1 | tail -15 > gpurun_out/r13_pytest.log
