python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_exp2.log 2>&1 || exit 1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_exp2.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_exp2.log
timeout 900 python scripts/sweep_env.py KVTC_C_GATHER_SIDE=0 KVTC_C_DEFLATE_SIDE=0 KVTC_C_GATHER_SIDE=0,KVTC_C_DEFLATE_SIDE=0 KVTC_GROUP_M_QUANT=2 --iters 10 > gpurun_out/sweep_exp2.log 2>&1; echo sweep rc=$?
grep sweep gpurun_out/sweep_exp2.log
