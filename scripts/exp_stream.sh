python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_exp16.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_codec.py tests/test_gpu_batch.py -x -q > gpurun_out/pytest_exp16.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_exp16.log | cut -c1-300
