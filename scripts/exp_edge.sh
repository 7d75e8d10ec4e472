python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_exp24.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_codec.py -x -q > gpurun_out/pytest_exp24.log 2>&1; echo "pytest rc=$?"; tail -25 gpurun_out/pytest_exp24.log | cut -c1-300
