timeout 1500 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -15 > gpurun_out/r8_pytest.log
timeout 300 python tools/time_config.py c3 5 > gpurun_out/r8_time_c3.log 2>&1
timeout 900 python tools/time_config.py c5 3 > gpurun_out/r8_time_c5.log 2>&1
