# round bench + evidence: bench lines (c3 default, c2, c4, c5), launch list, ncu --set full of the top kernel
set -x
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/b_c3.json 2> gpurun_out/b_c3.err
timeout 600 python bench.py --config c2 --steps 10 --warmup 3 > gpurun_out/b_c2.json 2> gpurun_out/b_c2.err
timeout 900 python bench.py --config c4 --steps 5 --warmup 3 > gpurun_out/b_c4.json 2> gpurun_out/b_c4.err
timeout 1500 python bench.py --config c5 --steps 5 --warmup 3 > gpurun_out/b_c5.json 2> gpurun_out/b_c5.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/b_ref_c3.json 2> gpurun_out/b_ref_c3.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c3.csv python tools/profile_once.py c3 > gpurun_out/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:msd_pass_kernel --launch-skip 5 --launch-count 1 -o gpurun_out/full_msd_pass python tools/profile_once.py c3 > gpurun_out/ncu_full1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:count_kernel --launch-skip 1 --launch-count 1 -o gpurun_out/full_count python tools/profile_once.py c3 > gpurun_out/ncu_full2.log 2>&1
