# final round evidence: full GPU suite + smoke, then tools/gpu_evidence.sh TAG
tag=${1:-r02e}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${tag}_build0.log 2>&1
timeout 1800 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -6 > gpurun_out/${tag}_gpu_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1
bash tools/gpu_evidence.sh $tag
