timeout 900 python -m pytest tests/test_parity.py -x -q -k "dd or c4 or fig1 or small or indexed or capacity or validation" 2>&1 | tail -15 > gpurun_out/r14_pytest.log
timeout 300 python tools/time_config.py c4 3 > gpurun_out/r14_time_c4.log 2>&1
