timeout 1200 python -m pytest tests/test_parity.py -x -q -k "msd or walk or fuzz or tie or small or c2_full" 2>&1 | tail -3 > gpurun_out/q_pytest.log
timeout 300 python tools/time_config.py c3 5 > gpurun_out/q_time_c3.log 2>&1
timeout 900 python tools/ab_flags.py c3 7 0 "ddm.DDM_COUNT_RANKS" > gpurun_out/ab.log 2>&1
