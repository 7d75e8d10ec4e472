#!/bin/bash
# Round-2 re-entry: verify the committed build on a B200 (GPU tests, smoke, bench) and run
# compute-sanitizer memcheck / racecheck once on the toy smoke.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02c.log 2>&1 || { tail -30 gpurun_out/build_r02c.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -rs > gpurun_out/pytest_gpu_r02c.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu_r02c.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_r02c.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke_r02c.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r02c.json 2> gpurun_out/bench_r02c.log; echo "bench rc=$?"; tail -c 600 gpurun_out/bench_r02c.json
for tool in memcheck racecheck synccheck; do
timeout 900 compute-sanitizer --tool $tool --print-limit 20 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/sanitizer_${tool}_r02c.log 2>&1; echo "sanitizer $tool rc=$?"; tail -4 gpurun_out/sanitizer_${tool}_r02c.log
done
