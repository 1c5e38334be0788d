# ncu of the big local sort (c5) -- run on the GPU box
timeout 900 ncu --set full --clock-control none --import-source on -k regex:local_sort_kernel --launch-skip 2 --launch-count 1 -o gpurun_out/p_lsbig python tools/profile_once.py c5 > gpurun_out/p_lsbig.log 2>&1
tail -2 gpurun_out/p_lsbig.log
