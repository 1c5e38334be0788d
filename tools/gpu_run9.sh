bash tools/gpu_quick.sh
timeout 600 ncu --set full --clock-control none --import-source on -k regex:local_sort_kernel --launch-skip 3 --launch-count 1 -o gpurun_out/r9_local_sort python tools/profile_once.py c3 > gpurun_out/r9_ncu1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:msd_pass_kernel --launch-skip 5 --launch-count 1 -o gpurun_out/r9_msd_pass python tools/profile_once.py c3 > gpurun_out/r9_ncu2.log 2>&1
