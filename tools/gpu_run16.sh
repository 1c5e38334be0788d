for i in 1 2; do
python tools/time_official.py c3 >> gpurun_out/r16.log 2>&1
python tools/time_official.py c5 3 >> gpurun_out/r16.log 2>&1
DDM_PASS_CTAS_PER_SM=3 python tools/time_official.py c5 3 >> gpurun_out/r16.log 2>&1
done
