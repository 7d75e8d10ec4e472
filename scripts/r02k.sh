#!/bin/bash
# Final-tree check (codec tests, smoke, bench line) + co-run CTA sweep of the overlapped schedule.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_k.log 2>&1 || { tail -30 gpurun_out/build_k.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_codec.py tests/test_gpu_stages.py -q -x > gpurun_out/pytest_k.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_k.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_k.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_k.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_k.json 2> gpurun_out/bench_k.log; echo "bench rc=$?"
python - gpurun_out/bench_k.json <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(round(d["value"], 2), round(d["ms_per_step"], 3), d["clocks"], d["roofline"]["frac"], d["step_ms_percentiles"])
PY
V="KVTC_CORUN_DEFLATE=1 KVTC_CORUN_GATHER=2 KVTC_CORUN_DEQUANT=1 KVTC_CORUN_DEFLATE=1,KVTC_CORUN_GATHER=2,KVTC_CORUN_DEQUANT=1"
timeout 1500 python scripts/sweep_env.py --iters 10 $V $V $V 2>&1 | grep sweep > gpurun_out/sweep_corun.log
python - <<'PY'
import re, collections
acc = collections.defaultdict(list)
for l in open("gpurun_out/sweep_corun.log"):
    m = re.match(r"\[sweep\] (\S+)\s+step=(\S+) ms", l)
    if m: acc[m.group(1)].append(float(m.group(2)))
for k, v in acc.items(): print(f"{k:70s} n={len(v)} mean={sum(v)/len(v):.3f} min={min(v):.2f} max={max(v):.2f}")
PY
