# short round-end evidence (one call, ~20 min): full GPU suite + smoke, ncu launch lists of
# c3 / c5 (traffic json refreshed), one ncu --set full capture of msd_hist_kernel turned into
# text on the box, then the bench lines of c3, c5, c4, c2 and the reference arm.
# usage: bash tools/gpu_final4.sh TAG
tag=$1
o=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $o/${tag}_build.log 2>&1
timeout 1500 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -6 > $o/${tag}_gpu_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > $o/${tag}_smoke.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,power.draw --format=csv > $o/${tag}_smi.csv
cp profiles/ncu_traffic.json $o/ncu_traffic.json
export DDM_SERIAL=1
for c in c3 c5; do
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 --csv \
    --log-file $o/${tag}_launches_$c.csv python tools/profile_once.py $c > $o/${tag}_ncu_launch_$c.log 2>&1
  n=$(grep -o "launches total: [0-9]*" $o/${tag}_ncu_launch_$c.log | awk '{print $3}')
  b=$(grep -o "launches before timed call: [0-9]*" $o/${tag}_ncu_launch_$c.log | awk '{print $5}')
  python tools/traffic_json.py $o/${tag}_launches_$c.csv $((n - b)) $c $o/ncu_traffic.json > $o/${tag}_traffic_$c.log 2>&1
  python tools/launches.py $o/${tag}_launches_$c.csv $((n - b)) > $o/${tag}_${c}_launch_summary.txt 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:msd_hist_kernel --launch-skip 3 --launch-count 1 -o $o/${tag}_msd_hist python tools/profile_once.py c3 > $o/${tag}_ncu1.log 2>&1
unset DDM_SERIAL
ncu -i $o/${tag}_msd_hist.ncu-rep --page details > $o/${tag}_msd_hist_ncu_full.txt 2>/dev/null
python tools/ncu_lines.py $o/${tag}_msd_hist.ncu-rep "" 30 > $o/${tag}_msd_hist_hot_lines.txt 2>/dev/null
rm -f $o/${tag}_msd_hist.ncu-rep
cp $o/ncu_traffic.json profiles/ncu_traffic.json
for c in c3 c5 c4 c2; do
  timeout 1200 python bench.py --config $c --steps 10 --warmup 3 > $o/${tag}_bench_$c.json 2> $o/${tag}_bench_$c.err
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $o/${tag}_bench_reference_c3.json 2> $o/${tag}_bench_reference_c3.err
