#!/bin/bash
# Branch-free DEFLATE emission (plain stores, edge words OR-ed after a barrier):
# parity + encoder time; A/B of the values' inflate beside the keys' GEMM.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_g.log 2>&1 || { tail -30 gpurun_out/build_g.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_stages.py tests/test_gpu_codec.py tests/test_gpu_batch.py tests/test_gpu_rans.py -x -q > gpurun_out/pytest_g.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_g.log
for rep in 1 2; do
for f in 0 1; do
KVTC_D_INFLATE_SIDE=$f timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_g_${f}_$rep.json 2> gpurun_out/bench_g_${f}_$rep.log
python - gpurun_out/bench_g_${f}_$rep.json <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
st = d.get("stages", {})
print(sys.argv[1], round(d.get("value"), 2), round(d.get("ms_per_step"), 3), (d.get("clocks") or {}).get("sm_mhz"), round(d["config"]["cr"], 3),
      {k: round(v.get("ms_per_step", 0), 3) for k, v in st.items() if k.startswith("d.") or k.startswith("c.")})
PY
done
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off -k "regex:deflate_encode|inflate|dequant" --csv --log-file gpurun_out/launches_g.csv python scripts/profile_run.py > /dev/null 2>&1
grep -E "deflate_encode|inflate|dequant" gpurun_out/launches_g.csv | awk -F'","' '{print $5, $NF}' | cut -c1-120
