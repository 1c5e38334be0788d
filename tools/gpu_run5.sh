timeout 1200 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -15 > gpurun_out/r5_pytest.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dd_tile_kernel --launch-skip 2 --launch-count 1 -o gpurun_out/r5_dd_count python tools/profile_once.py c4 > gpurun_out/r5_ncu.log 2>&1
