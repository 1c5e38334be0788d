bash tools/gpu_quick.sh
DDM_PASS_CTAS_PER_SM=1 timeout 300 python tools/time_config.py c3 5 > gpurun_out/q_time_c3_cap1.log 2>&1
DDM_PASS_CTAS_PER_SM=2 timeout 300 python tools/time_config.py c3 5 > gpurun_out/q_time_c3_cap2.log 2>&1
