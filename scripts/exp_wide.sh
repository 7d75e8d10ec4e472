python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_exp22.log 2>&1 || exit 1
timeout 1200 python -m pytest tests/test_gpu_codec.py tests/test_gpu_fullscale.py -x -q > gpurun_out/pytest_exp22.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_exp22.log | cut -c1-300
timeout 1200 python scripts/sweep_env.py KVTC_C_DEFLATE_SIDE=0 --iters 10 > gpurun_out/sweep_exp22.log 2>&1; echo sweep rc=$?
grep sweep gpurun_out/sweep_exp22.log | cut -c1-330
