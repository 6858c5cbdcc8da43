python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fc_smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/fc_pytest.log 2>&1; echo pytest=$?
timeout 900 python bench.py > gpurun_out/fc_bench.json 2> gpurun_out/fc_bench.err; echo bench=$?
