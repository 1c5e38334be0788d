# bench lines for every config + the reference arm (c3)
for c in c3 c2 c4 c5; do timeout 1500 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/b_$c.json 2> gpurun_out/b_$c.err; done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/b_ref_c3.json 2> gpurun_out/b_ref_c3.err
