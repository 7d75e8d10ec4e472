python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_exp8.log 2>&1 || exit 1
timeout 2400 python -m pytest tests -m gpu -x -q -s -k "configs" > gpurun_out/pytest_exp8.log 2>&1; echo "pytest configs rc=$?"; grep -E "passed|failed|nemo12b|llama70b|Error|error" gpurun_out/pytest_exp8.log | tail -12
timeout 900 python bench.py --config multiconv --convs 24 --steps 1 --warmup 1 > gpurun_out/bench_mc.json 2> gpurun_out/bench_mc.log; echo "multiconv rc=$?"; cat gpurun_out/bench_mc.json | cut -c1-600; tail -3 gpurun_out/bench_mc.log
KVTC_QUANT_NSUB=2 timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:gemm -c 1 -o gpurun_out/prof_nsub2 -f python scripts/profile_run.py > /dev/null 2>&1; echo "ncu nsub2 rc=$?"
python scripts/ncu_hotlines.py gpurun_out/prof_nsub2.ncu-rep gemm_kernel 40 > gpurun_out/hot_nsub2.txt 2>&1; head -30 gpurun_out/hot_nsub2.txt
rm -f gpurun_out/prof_nsub2.ncu-rep
