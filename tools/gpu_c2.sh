# c2: official-style timing + per-kernel profile, launch list, ncu of the chunk emit (run on the GPU box)
timeout 300 python tools/variant_time.py c2 20 > gpurun_out/c2_time.jsonl 2>gpurun_out/c2_time.err
DDM_SERIAL=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/c2_launches.csv python tools/profile_once.py c2 > gpurun_out/c2_ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:emit_chunk --launch-skip 1 --launch-count 1 -o gpurun_out/p_emit_chunk python tools/profile_once.py c2 > gpurun_out/p_ec.log 2>&1
tail -2 gpurun_out/p_ec.log
