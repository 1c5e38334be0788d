# bench lines only (after a profiles/ncu_traffic.json update); args: TAG configs...
tag=$1; shift
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${tag}_build.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,power.draw --format=csv > gpurun_out/${tag}_smi.csv
for c in "$@"; do
  timeout 1500 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/${tag}_bench_$c.json 2> gpurun_out/${tag}_bench_$c.err
done
for a in 0.01 1 100; do
  timeout 900 python bench.py --config c3 --mode count --alpha $a --steps 10 --warmup 3 > gpurun_out/${tag}_bench_c3_count_a$a.json 2> gpurun_out/${tag}_bench_c3_count_a$a.err
done
