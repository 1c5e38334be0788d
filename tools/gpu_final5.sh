# the remaining bench lines at the final tree: c1 and the count-mode alpha sweep.  usage: bash tools/gpu_final5.sh TAG
tag=$1; o=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $o/${tag}_build5.log 2>&1
timeout 600 python bench.py --config c1 --steps 10 --warmup 3 > $o/${tag}_bench_c1.json 2> $o/${tag}_bench_c1.err
for a in 0.01 1 100; do
  timeout 600 python bench.py --config c3 --mode count --alpha $a --steps 10 --warmup 3 > $o/${tag}_bench_c3_count_a$a.json 2> $o/${tag}_bench_c3_count_a$a.err
done
