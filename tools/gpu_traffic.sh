# ncu launch lists (time + DRAM bytes) for c2 and c5, then their bench lines
export DDM_SERIAL=1
for c in c2 c5; do
  timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/f_launches_$c.csv python tools/profile_once.py $c > gpurun_out/f_ncu_launch_$c.log 2>&1
done
