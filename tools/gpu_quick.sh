# quick check: sort/match parity subset + c3 timing (args: extra configs to time)
timeout 900 python -m pytest tests/test_parity.py -x -q -k "msd or walk or fuzz or c1 or c2_full or ragged or long or clamped or small or tie or dd_chunks or c5_scaled or validation or capacity or empty or asymmetric or extreme" 2>&1 | tail -4 > gpurun_out/q_pytest.log
timeout 300 python tools/time_config.py c3 5 > gpurun_out/q_time_c3.log 2>&1
for c in "$@"; do timeout 600 python tools/time_config.py $c 3 > gpurun_out/q_time_$c.log 2>&1; done
