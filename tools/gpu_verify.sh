# verify HEAD on one B200: full GPU suite + smoke, c3 pairs and count-mode bench lines
tag=${1:-r02g}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${tag}_build.log 2>&1
timeout 1800 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -8 > gpurun_out/${tag}_gpu_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1
timeout 900 python bench.py --config c3 --steps 10 --warmup 3 > gpurun_out/${tag}_bench_c3.json 2> gpurun_out/${tag}_bench_c3.err
for a in 0.01 1 100; do
  timeout 900 python bench.py --config c3 --mode count --alpha $a --steps 10 --warmup 3 > gpurun_out/${tag}_bench_c3_count_a$a.json 2> gpurun_out/${tag}_bench_c3_count_a$a.err
done
