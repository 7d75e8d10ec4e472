#!/bin/bash
# A/B of the codec schedule after the codec-kernel rewrites: side stream beside the
# GEMMs (default) vs every kernel on the caller's stream (KVTC_NO_OVERLAP=1), interleaved.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_j.log 2>&1 || { tail -30 gpurun_out/build_j.log; exit 1; }
for rep in 1 2 3; do
for f in 0 1; do
if [ $f = 1 ]; then export KVTC_NO_OVERLAP=1; else unset KVTC_NO_OVERLAP; fi
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_j_${f}_$rep.json 2> gpurun_out/bench_j_${f}_$rep.log
python - gpurun_out/bench_j_${f}_$rep.json <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
st = d.get("stages", {})
print(sys.argv[1], round(d.get("value"), 2), round(d.get("ms_per_step"), 3), (d.get("clocks") or {}).get("sm_mhz"),
      d["step_ms_percentiles"], {k: round(v.get("ms_per_step", 0), 2) for k, v in st.items() if "gemm" in k})
PY
done
done
unset KVTC_NO_OVERLAP
