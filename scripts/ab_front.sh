#!/bin/bash
# A/B of the decompression front end: one inflate+dequantise launch (default) vs
# the inflater followed by the dequantiser (KVTC_D_INFLATE_DQ=0), interleaved.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_ab.log 2>&1 || { tail -30 gpurun_out/build_ab.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_codec.py -x -q -k "front_end or vs_oracle" > gpurun_out/pytest_ab.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_ab.log
for rep in 1 2; do
for f in 1 0; do
KVTC_D_INFLATE_DQ=$f timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_ab_${f}_$rep.json 2> gpurun_out/bench_ab_${f}_$rep.log
python - gpurun_out/bench_ab_${f}_$rep.json <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
st = d.get("stages", {})
print(sys.argv[1], round(d.get("value"), 2), round(d.get("ms_per_step"), 3), (d.get("clocks") or {}).get("sm_mhz"),
      {k: round(v.get("ms_per_step", 0), 3) for k, v in st.items() if k.startswith("d.") or k in ("c.deflate",)})
PY
done
done
for f in 1 0; do
KVTC_D_INFLATE_DQ=$f timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off -k "regex:inflate|dequant" --csv --log-file gpurun_out/launches_ab_$f.csv python scripts/profile_run.py > /dev/null 2>&1
grep -E "inflate|dequant" gpurun_out/launches_ab_$f.csv | awk -F'","' -v f=$f '{print f, $5, $NF}' | cut -c1-160
done
