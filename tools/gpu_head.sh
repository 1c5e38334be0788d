# HEAD check on one B200: full GPU suite, smoke, per-config timings with phase breakdown
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/h_build.log 2>&1
timeout 1800 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -15 > gpurun_out/h_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/h_smoke.log 2>&1
for c in c3 c4 c5 c2; do timeout 600 python tools/time_config.py $c 5 > gpurun_out/h_time_$c.log 2>&1; done
