python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_exp25.log 2>&1 || exit 1
KVTC_D_INFLATE_SIDE=1 timeout 900 python -m pytest tests/test_gpu_codec.py -x -q > gpurun_out/pytest_exp25.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_exp25.log | cut -c1-200
timeout 1500 python scripts/sweep_env.py KVTC_D_INFLATE_SIDE=1 KVTC_D_INFLATE_SIDE=1,KVTC_CORUN_INFLATE=1 KVTC_D_INFLATE_SIDE=1 --iters 10 > gpurun_out/sweep_exp25.log 2>&1; echo sweep rc=$?
grep sweep gpurun_out/sweep_exp25.log | sed 's/c.raw_tokens.*d.inflate/... d.inflate/' | cut -c1-260
