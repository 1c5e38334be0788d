timeout 900 python -m pytest tests/test_parity.py -x -q -k "dd or c4 or capacity or indexed or slab or fuzz" 2>&1 | tail -2 > gpurun_out/q_pytest.log
DDM_SERIAL=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:dd_tile_kernel --launch-skip 1 --launch-count 1 -o gpurun_out/f_dd_stage python tools/profile_once.py c4 > gpurun_out/f_ncu5.log 2>&1
