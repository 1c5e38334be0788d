timeout 900 python -m pytest tests/test_parity.py -x -q -k "walk or fuzz or long or c2_full or c3_full or small or tie or asymmetric or extreme" 2>&1 | tail -3 > gpurun_out/q_pytest.log
timeout 900 python tools/ab_flags.py c2,c3,c5 7 0 "ddm.DDM_COUNT_RANKS" > gpurun_out/ab.log 2>&1
timeout 300 python tools/time_config.py c3 5 > gpurun_out/q_time_c3.log 2>&1
