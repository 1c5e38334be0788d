# d > 1 filter forms: parity tests, then c4 timing of both forms (run on the GPU box)
timeout 900 python -m pytest tests/test_parity.py -x -q -k "dd or c4 or sweep_dim or literal" > gpurun_out/dd_pytest.log 2>&1
tail -3 gpurun_out/dd_pytest.log
timeout 300 python tools/variant_time.py c4 7 > gpurun_out/dd_c4.jsonl 2>gpurun_out/dd_c4.err
DDM_DD_CHUNKS=1 timeout 300 python tools/variant_time.py c4 7 >> gpurun_out/dd_c4.jsonl 2>>gpurun_out/dd_c4.err
tail -c 1500 gpurun_out/dd_c4.err
