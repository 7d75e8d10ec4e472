#!/bin/bash
# Round-2 measurement session: new parity tests, then the BASELINE configs as bench lines.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02b.log 2>&1 || { tail -30 gpurun_out/build_r02b.log; exit 1; }
timeout 1500 python -m pytest tests/test_gpu_calib_dp.py tests/test_gpu_batch.py tests/test_gpu_codec.py -m gpu -q -rs -s > gpurun_out/pytest_r02b.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_r02b.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r02b.json 2> gpurun_out/bench_r02b.log; echo "bench llama8b rc=$?"
timeout 900 python bench.py --config llama70b_shard --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_r02b_70b.json 2> gpurun_out/bench_r02b_70b.log; echo "bench 70b rc=$?"
for cr in 8 16 32; do
timeout 900 python bench.py --config nemo12b --cr $cr --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_r02b_nemo_cr$cr.json 2> gpurun_out/bench_r02b_nemo_cr$cr.log; echo "bench nemo cr$cr rc=$?"
done
timeout 1800 python bench.py --config multiconv --steps 1 --warmup 1 > gpurun_out/bench_r02b_mc256.json 2> gpurun_out/bench_r02b_mc256.log; echo "bench multiconv rc=$?"
for f in gpurun_out/bench_r02b*.json; do python - "$f" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[1], round(d["value"], 2), d.get("ms_per_step"), d.get("clocks", {}).get("sm_mhz"), d["config"].get("cr"), d["config"].get("r_eff"))
except Exception as e:
    print(sys.argv[1], "ERR", e)
PY
done
