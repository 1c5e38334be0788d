# Copy one evidence run (tools/gpu_evidence.sh TAG) from gpurun_out/ into profiles/ as
# text: bench lines, launch-list summaries, ncu details pages and hot source lines.
# usage: bash tools/collect_profiles.sh TAG OUT_PREFIX   (e.g. r02b r02)
tag=$1; out=${2:-r02}
o=gpurun_out; p=profiles
for f in $o/${tag}_bench_*.json; do b=$(basename $f .json); cp $f $p/${out}_${b#${tag}_}.json; done
cp $o/${tag}_launches_c3.csv $p/${out}_c3_launches_serialised.csv
for c in c2 c3 c4 c5; do
  n=$(grep -o "launches total: [0-9]*" $o/${tag}_ncu_launch_$c.log | awk '{print $3}')
  b=$(grep -o "launches before timed call: [0-9]*" $o/${tag}_ncu_launch_$c.log | awk '{print $5}')
  { echo "# ncu launch list of the last pairs call of DDM_SERIAL=1 tools/profile_once.py $c (gpu__time_duration, DRAM bytes; serialised, cold)";
    python tools/launches.py $o/${tag}_launches_$c.csv $((n - b)); } > $p/${out}_${c}_launch_summary.txt
done
for k in msd_pass local_sort count emit dd_stage; do
  if [ -d $o/${tag}_prof ]; then  # (tools/gpu_final3.sh: reports already turned into text on the box)
    cp $o/${tag}_prof/${k}_ncu_full.txt $p/${out}_${k}_ncu_full.txt 2>/dev/null
    cp $o/${tag}_prof/${k}_hot_lines.txt $p/${out}_${k}_hot_lines.txt 2>/dev/null
    continue
  fi
  [ -f $o/${tag}_$k.ncu-rep ] || continue
  ncu -i $o/${tag}_$k.ncu-rep --page details > $p/${out}_${k}_ncu_full.txt 2>/dev/null
  python tools/ncu_lines.py $o/${tag}_$k.ncu-rep "" 30 > $p/${out}_${k}_hot_lines.txt 2>/dev/null
done
cp $o/${tag}_smi.csv $p/${out}_smi.csv 2>/dev/null
ls -la $p | grep $out
