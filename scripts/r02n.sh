#!/bin/bash
# rANS back-end: parity (GPU == oracle streams, decode of oracle sections) and bench line.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02n.log 2>&1 || { tail -30 gpurun_out/build_r02n.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_rans.py tests/test_gpu_codec.py -m gpu -x -q -s -k "rans" > gpurun_out/pytest_r02n.log 2>&1; echo "tests rc=$?"; tail -4 gpurun_out/pytest_r02n.log; grep "\[rans\]" gpurun_out/pytest_r02n.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --coder rans > gpurun_out/bench_r02n_rans.json 2> gpurun_out/bench_r02n_rans.log; echo "bench rans rc=$?"
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_r02n_rans.json").read().strip().splitlines()[-1])
print(round(d["value"], 2), round(d["ms_per_step"], 2), d["clocks"]["sm_mhz"], round(d["config"]["cr"], 3))
for k in ("c.rans_keys", "c.rans_values_overlapped", "d.rans_decode"):
    print(k, d["stages"].get(k))
PY
