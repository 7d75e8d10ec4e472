#!/bin/bash
# Round-2 final validation (fifth pass: final tree, values inflate beside the keys GEMM): GPU suite, smoke, bench lines of the BASELINE configs, ncu launch list + summary.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_f5.log 2>&1 || { tail -30 gpurun_out/build_f5.log; exit 1; }
timeout 1800 python -m pytest tests -m gpu -q -rs -s > gpurun_out/pytest_gpu_f5.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed" gpurun_out/pytest_gpu_f5.log | tail -2
grep -E "^\[codes\]|\[joint\]|\[rans\]" gpurun_out/pytest_gpu_f5.log > gpurun_out/codes_f5.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_f5.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_f5.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_f5.json 2> gpurun_out/bench_f5.log; echo "bench rc=$?"
timeout 900 python bench.py --config llama70b_shard --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_f5_70b.json 2> gpurun_out/bench_f5_70b.log; echo "bench 70b rc=$?"
for cr in 8 16 32; do
timeout 900 python bench.py --config nemo12b --cr $cr --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_f5_nemo$cr.json 2> gpurun_out/bench_f5_nemo$cr.log; echo "bench nemo cr$cr rc=$?"
done
timeout 1800 python bench.py --config multiconv --steps 1 --warmup 1 > gpurun_out/bench_f5_mc256.json 2> gpurun_out/bench_f5_mc256.log; echo "bench multiconv rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_f5_ref.json 2> gpurun_out/bench_f5_ref.log; echo "bench ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_f5.csv python scripts/profile_run.py > gpurun_out/launches_f5.log 2>&1; echo "launches rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on --profile-from-start off -k "regex:gemm_kernel|deflate_encode|inflate_fast|dequant_rows|gather_kernel" -o gpurun_out/prof_f5 -f python scripts/profile_run.py > gpurun_out/full_f5.log 2>&1; echo "full rc=$?"
python scripts/ncu_summary.py gpurun_out/launches_f5.csv gpurun_out/prof_f5.ncu-rep gpurun_out/summary_f5.md gpurun_out/traffic_f5.json r02_final5 > /dev/null 2>&1; echo "summary rc=$?"
rm -f gpurun_out/prof_f5.ncu-rep
for f in gpurun_out/bench_f5*.json; do python - "$f" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[1], d.get("value"), d.get("ms_per_step"), (d.get("clocks") or {}).get("sm_mhz"), (d.get("config") or {}).get("cr"))
except Exception as e:
    print(sys.argv[1], "ERR", e)
PY
done
