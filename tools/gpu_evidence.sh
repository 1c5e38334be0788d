# Round evidence on one B200 (run from the repo root under gpurun): ncu launch lists
# (per-phase DRAM traffic -> gpurun_out/ncu_traffic.json, copied to profiles/ for the
# bench's roofline.traffic), ncu full captures of the dominant kernels, then the bench
# lines of every config, the reference arm, the count-mode alpha sweep and the
# multi-GPU path on one GPU (gloo).   usage: bash tools/gpu_evidence.sh TAG
tag=${1:-r02d}
o=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $o/${tag}_build.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,power.draw --format=csv > $o/${tag}_smi.csv
export DDM_SERIAL=1
for c in c3 c2 c5 c4; do
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 --csv \
    --log-file $o/${tag}_launches_$c.csv python tools/profile_once.py $c > $o/${tag}_ncu_launch_$c.log 2>&1
  n=$(grep -o "launches total: [0-9]*" $o/${tag}_ncu_launch_$c.log | awk '{print $3}')
  b=$(grep -o "launches before timed call: [0-9]*" $o/${tag}_ncu_launch_$c.log | awk '{print $5}')
  python tools/traffic_json.py $o/${tag}_launches_$c.csv $((n - b)) $c $o/ncu_traffic.json > $o/${tag}_traffic_$c.log 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:msd_pass_kernel --launch-skip 7 --launch-count 1 -o $o/${tag}_msd_pass python tools/profile_once.py c3 > $o/${tag}_ncu1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:local_sort_kernel --launch-skip 3 --launch-count 1 -o $o/${tag}_local_sort python tools/profile_once.py c3 > $o/${tag}_ncu2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:count_kernel --launch-skip 1 --launch-count 1 -o $o/${tag}_count python tools/profile_once.py c3 > $o/${tag}_ncu3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:emit_tile --launch-skip 0 --launch-count 1 -o $o/${tag}_emit python tools/profile_once.py c3 > $o/${tag}_ncu4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rows_kernel --launch-skip 1 --launch-count 1 -o $o/${tag}_dd_stage python tools/profile_once.py c4 > $o/${tag}_ncu5.log 2>&1
timeout 900 ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum --clock-control none -k regex:rows_kernel --csv --log-file $o/${tag}_dd_inst.csv python tools/profile_once.py c4 > $o/${tag}_ncu6.log 2>&1
unset DDM_SERIAL
python tools/inst_json.py $o/${tag}_dd_inst.csv $o/ncu_inst.json > $o/${tag}_inst.log 2>&1
cp $o/ncu_traffic.json profiles/ncu_traffic.json
cp $o/ncu_inst.json profiles/ncu_inst.json
for c in c3 c1 c2 c4 c5; do
  timeout 1500 python bench.py --config $c --steps 10 --warmup 3 > $o/${tag}_bench_$c.json 2> $o/${tag}_bench_$c.err
done
for a in 0.01 1 100; do
  timeout 900 python bench.py --config c3 --mode count --alpha $a --steps 10 --warmup 3 > $o/${tag}_bench_c3_count_a$a.json 2> $o/${tag}_bench_c3_count_a$a.err
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $o/${tag}_bench_reference_c3.json 2> $o/${tag}_bench_reference_c3.err
timeout 900 python bench.py --gpus 2 --backend gloo --config c3 --steps 3 --warmup 3 > $o/${tag}_bench_c3_g2_gloo.json 2> $o/${tag}_bench_c3_g2_gloo.err
timeout 900 python bench.py --gpus 2 --backend gloo --dist broadcast --config c3 --steps 3 --warmup 3 > $o/${tag}_bench_c3_g2_gloo_bc.json 2> $o/${tag}_bench_c3_g2_gloo_bc.err
