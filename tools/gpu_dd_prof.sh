# d > 1: parity tests, c4 timing, ncu of the row-indexed stage pass (run on the GPU box)
bash tools/gpu_dd.sh
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rows_kernel --launch-skip 1 --launch-count 1 -o gpurun_out/p_rows3 python tools/profile_once.py c4 > gpurun_out/p_rows3.log 2>&1
tail -2 gpurun_out/p_rows3.log
