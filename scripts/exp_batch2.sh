python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_exp11.log 2>&1 || { tail -20 gpurun_out/build_exp11.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_batch.py tests/test_gpu_codec.py -x -q > gpurun_out/pytest_exp11.log 2>&1; echo "pytest batch rc=$?"; tail -5 gpurun_out/pytest_exp11.log | cut -c1-300
timeout 1200 python bench.py --config multiconv --convs 32 --steps 1 --warmup 1 > gpurun_out/bench_mc2.json 2> gpurun_out/bench_mc2.log; echo "multiconv rc=$?"; cut -c1-500 gpurun_out/bench_mc2.json; tail -3 gpurun_out/bench_mc2.log
