DDM_SERIAL=1 timeout 300 python tools/time_config.py c3 5 > gpurun_out/q_time_c3_serial.log 2>&1
