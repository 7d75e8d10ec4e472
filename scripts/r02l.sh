#!/bin/bash
# Round-2 validation: full GPU suite (with -s for the per-type code-parity lines), smoke, bench, launch list, ncu of the codec kernels.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02l.log 2>&1 || { tail -30 gpurun_out/build_r02l.log; exit 1; }
timeout 1800 python -m pytest tests -m gpu -q -rs -s > gpurun_out/pytest_gpu_r02l.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed" gpurun_out/pytest_gpu_r02l.log | tail -2
grep -E "^\[codes\]|\[joint\]" gpurun_out/pytest_gpu_r02l.log > gpurun_out/codes_r02l.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_r02l.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_r02l.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r02l.json 2> gpurun_out/bench_r02l.log; echo "bench rc=$?"; tail -c 300 gpurun_out/bench_r02l.json
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --chunk-bytes 32768 > gpurun_out/bench_r02l_c32k.json 2> gpurun_out/bench_r02l_c32k.log; echo "bench c32k rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_r02l.csv python scripts/profile_run.py > gpurun_out/launches_r02l.log 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k "regex:gemm_kernel|deflate_encode|inflate_fast|dequant_kernel|gather_kernel" -o gpurun_out/prof_r02l -f python scripts/profile_run.py > gpurun_out/full_r02l.log 2>&1; echo "full rc=$?"
python scripts/ncu_summary.py gpurun_out/launches_r02l.csv gpurun_out/prof_r02l.ncu-rep gpurun_out/summary_r02l.md gpurun_out/traffic_r02l.json r02l > /dev/null 2>&1; echo "summary rc=$?"
for k in "deflate_encode" "inflate_fast"; do echo "== $k"; python scripts/ncu_hotlines.py gpurun_out/prof_r02l.ncu-rep "$k" 20 1; done > gpurun_out/hotlines_r02l.txt 2>&1
rm -f gpurun_out/prof_r02l.ncu-rep
