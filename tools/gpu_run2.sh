set -x
free -g; nproc
timeout 300 python tools/time_config.py c4 2 > gpurun_out/r2_time_c4.log 2>&1
timeout 900 python tools/time_config.py c5 3 > gpurun_out/r2_time_c5.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:msd_pass_kernel --launch-skip 5 --launch-count 1 -o gpurun_out/r2_msd_pass python tools/profile_once.py c3 > gpurun_out/r2_ncu1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:local_sort_kernel --launch-skip 3 --launch-count 1 -o gpurun_out/r2_local_sort python tools/profile_once.py c3 > gpurun_out/r2_ncu2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:count_kernel --launch-skip 1 --launch-count 1 -o gpurun_out/r2_count python tools/profile_once.py c3 > gpurun_out/r2_ncu3.log 2>&1
