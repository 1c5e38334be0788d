set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/r1_pytest.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r1_bench_c3.json 2> gpurun_out/r1_bench_c3.err
timeout 600 python bench.py --config c2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r1_bench_c2.json 2> gpurun_out/r1_bench_c2.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/r1_launches_c3.csv python tools/profile_once.py c3 > gpurun_out/r1_ncu.log 2>&1
python tools/launches.py gpurun_out/r1_launches_c3.csv 60 > gpurun_out/r1_launch_summary.txt 2>&1
