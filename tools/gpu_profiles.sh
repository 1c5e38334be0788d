# ncu evidence with the sort chains serialised (DDM_SERIAL=1: the configuration of bench.py's profiled region)
export DDM_SERIAL=1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/p_launches_c3.csv python tools/profile_once.py c3 > gpurun_out/p_ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:msd_pass_kernel --launch-skip 5 --launch-count 1 -o gpurun_out/p_msd_pass python tools/profile_once.py c3 > gpurun_out/p_ncu1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:local_sort_kernel --launch-skip 3 --launch-count 1 -o gpurun_out/p_local_sort python tools/profile_once.py c3 > gpurun_out/p_ncu2.log 2>&1
