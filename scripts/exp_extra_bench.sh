python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_extra.log 2>&1 || exit 1
timeout 1500 python bench.py --config nemo12b --tokens 65536 --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_nemo.json 2> gpurun_out/bench_nemo.log; echo "nemo rc=$?"; cut -c1-400 gpurun_out/bench_nemo.json
timeout 1500 python bench.py --config multiconv --convs 64 --steps 1 --warmup 1 > gpurun_out/bench_mc64.json 2> gpurun_out/bench_mc64.log; echo "multiconv rc=$?"; cut -c1-400 gpurun_out/bench_mc64.json
