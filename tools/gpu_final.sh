# round-end evidence: bench lines, launch list (c3), ncu full of the dominant kernels
set -x
for c in c3 c2 c4 c5; do timeout 1500 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/f_b_$c.json 2> gpurun_out/f_b_$c.err; done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/f_b_ref_c3.json 2> gpurun_out/f_b_ref_c3.err
export DDM_SERIAL=1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/f_launches_c3.csv python tools/profile_once.py c3 > gpurun_out/f_ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:msd_pass_kernel --launch-skip 7 --launch-count 1 -o gpurun_out/f_msd_pass python tools/profile_once.py c3 > gpurun_out/f_ncu1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:local_sort_kernel --launch-skip 3 --launch-count 1 -o gpurun_out/f_local_sort python tools/profile_once.py c3 > gpurun_out/f_ncu2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:count_kernel --launch-skip 1 --launch-count 1 -o gpurun_out/f_count python tools/profile_once.py c3 > gpurun_out/f_ncu3.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:emit_tile --launch-skip 0 --launch-count 1 -o gpurun_out/f_emit python tools/profile_once.py c3 > gpurun_out/f_ncu4.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dd_tile_kernel --launch-skip 1 --launch-count 1 -o gpurun_out/f_dd_stage python tools/profile_once.py c4 > gpurun_out/f_ncu5.log 2>&1
