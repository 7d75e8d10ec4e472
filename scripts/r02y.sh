#!/bin/bash
# Inflate decode-loop rewrite + 11-bit code limit: parity, bench A/B (limit 11 vs 15), codec kernel times.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_y.log 2>&1 || { tail -30 gpurun_out/build_y.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_stages.py tests/test_gpu_codec.py tests/test_gpu_integrity.py tests/test_gpu_batch.py -x -q > gpurun_out/pytest_y.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_y.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_y11.json 2> gpurun_out/bench_y11.log; echo "bench11 rc=$?"
KVTC_DEFLATE_MAXBITS=15 timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_y15.json 2> gpurun_out/bench_y15.log; echo "bench15 rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off -k "regex:inflate_fast|deflate_encode|dequant_kernel" --csv --log-file gpurun_out/launches_y.csv python scripts/profile_run.py > gpurun_out/launches_y.log 2>&1; echo "ncu rc=$?"
for f in gpurun_out/bench_y*.json; do python - "$f" <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
st = d.get("stages", {})
print(sys.argv[1], d.get("value"), d.get("ms_per_step"), (d.get("clocks") or {}).get("sm_mhz"), (d.get("config") or {}).get("cr"),
      {k: round(v.get("ms_per_step", 0), 3) for k, v in st.items() if k in ("d.inflate", "d.dequant", "c.deflate")})
PY
done
grep -E "inflate_fast|deflate_encode|dequant_kernel" gpurun_out/launches_y.csv | awk -F'","' '{print $5, $NF}' | head
