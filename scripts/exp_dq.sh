python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_exp26.log 2>&1 || exit 1
timeout 1200 python -m pytest tests/test_gpu_stages.py tests/test_gpu_codec.py tests/test_gpu_fullscale.py tests/test_gpu_batch.py -x -q > gpurun_out/pytest_exp26.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_exp26.log | cut -c1-200
timeout 600 ncu --metrics gpu__time_duration.sum -k regex:dequant --profile-from-start off --clock-control none --csv --log-file gpurun_out/ncu_exp26.csv python scripts/profile_run.py > /dev/null 2>&1
grep -E "dequant" gpurun_out/ncu_exp26.csv | awk -F'","' '{print $5, $NF}' | cut -c1-120
