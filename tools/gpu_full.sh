# full GPU suite + c2/c3/c4 timing (run on the GPU box)
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/full_pytest.log 2>&1
tail -3 gpurun_out/full_pytest.log
for c in c2 c3 c4; do timeout 300 python tools/variant_time.py $c 10 >> gpurun_out/full_time.jsonl 2>>gpurun_out/full_time.err; done
