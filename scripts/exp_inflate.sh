python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_exp17.log 2>&1 || exit 1
timeout 1200 python -m pytest tests/test_gpu_stages.py tests/test_gpu_codec.py tests/test_gpu_batch.py tests/test_gpu_fullscale.py -x -q > gpurun_out/pytest_exp17.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_exp17.log | cut -c1-300
timeout 900 python scripts/sweep_env.py --iters 10 > gpurun_out/sweep_exp17.log 2>&1; echo sweep rc=$?
grep sweep gpurun_out/sweep_exp17.log | cut -c1-330
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum -k regex:inflate --profile-from-start off --clock-control none --csv --log-file gpurun_out/ncu_exp17.csv python scripts/profile_run.py > /dev/null 2>&1
grep -E "inflate" gpurun_out/ncu_exp17.csv | cut -c1-80,200-400
