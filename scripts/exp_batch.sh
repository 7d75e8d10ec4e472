python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_exp10.log 2>&1 || { tail -20 gpurun_out/build_exp10.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_batch.py -x -q > gpurun_out/pytest_exp10.log 2>&1; echo "pytest batch rc=$?"; tail -30 gpurun_out/pytest_exp10.log | cut -c1-300
timeout 1500 python -m pytest tests -m gpu -x -q -k "not configs and not batch" > gpurun_out/pytest_exp10b.log 2>&1; echo "pytest rest rc=$?"; tail -3 gpurun_out/pytest_exp10b.log
