timeout 1500 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -4 > gpurun_out/r10_pytest.log
timeout 300 python tools/time_config.py c3 5 > gpurun_out/r10_time_c3.log 2>&1
DDM_PASS_CTAS_PER_SM=2 timeout 300 python tools/time_config.py c3 5 > gpurun_out/r10_time_c3_cap2.log 2>&1
DDM_PASS_CTAS_PER_SM=1 timeout 300 python tools/time_config.py c3 5 > gpurun_out/r10_time_c3_cap1.log 2>&1
timeout 300 python tools/time_config.py c2 5 > gpurun_out/r10_time_c2.log 2>&1
