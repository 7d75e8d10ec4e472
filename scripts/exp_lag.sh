python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_exp12.log 2>&1 || { tail -20 gpurun_out/build_exp12.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_calib_dp.py -x -q > gpurun_out/pytest_exp12.log 2>&1; echo "pytest dp rc=$?"; tail -3 gpurun_out/pytest_exp12.log | cut -c1-300
timeout 1200 python scripts/sweep_env.py KVTC_SYNC_LAG_QUANT=1 KVTC_GROUP_M_QUANT=8 KVTC_GROUP_M_QUANT=16 KVTC_GROUP_M_QUANT=8,KVTC_SYNC_LAG_QUANT=1 --iters 10 > gpurun_out/sweep_exp12.log 2>&1; echo sweep rc=$?
grep sweep gpurun_out/sweep_exp12.log | cut -c1-200
