timeout 900 python -m pytest tests/test_parity.py -x -q -k "c2 or small or fuzz or tie or chunk or dense or capacity or long or walk" > gpurun_out/q2_pytest.log 2>&1
tail -2 gpurun_out/q2_pytest.log
rm -f gpurun_out/q2_time.jsonl
for c in c2 c3; do timeout 300 python tools/variant_time.py $c 10 >> gpurun_out/q2_time.jsonl 2>>gpurun_out/q2_time.err; done
