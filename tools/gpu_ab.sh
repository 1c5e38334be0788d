timeout 1200 python -m pytest tests/test_parity.py -x -q -k "walk or fuzz or long or c2_full or c3_full or c5_full or small or tie or asymmetric or extreme or capacity or graph or pipelined or msd or slab or indexed or empty or ragged" 2>&1 | tail -5 > gpurun_out/q_pytest.log
timeout 900 python tools/ab_flags.py c1,c2,c3,c5 7 0 "ddm.DDM_COUNT_RANKS" "ddm.DDM_COUNT_WALK|ddm.DDM_EMIT_FORCE_CHUNK" > gpurun_out/ab.log 2>&1
timeout 300 python tools/time_config.py c3 5 > gpurun_out/q_time_c3.log 2>&1
