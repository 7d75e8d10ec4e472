python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_fc.log 2>&1 || exit 1
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_fc.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/smoke_fc.log
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.log; echo "ref rc=$?"; cut -c1-600 gpurun_out/bench_ref.json
