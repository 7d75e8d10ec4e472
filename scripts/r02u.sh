#!/bin/bash
# A/B of the compress-GEMM slowdown between e0b4133 (_ab/old, built here) and HEAD on
# one box: alternating bench runs, then env-knob variants of HEAD in one process.
mkdir -p gpurun_out
R=$PWD
timeout 900 python -m pytest tests/test_gpu_stages.py tests/test_gpu_codec.py -m gpu -x -q 2>&1 | tail -3; echo "tests rc=$?"
for i in 1 2; do
  (cd _ab/old && timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu > $R/gpurun_out/ab_old$i.json 2> $R/gpurun_out/ab_old$i.log); echo "old$i rc=$?"
  timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/ab_new$i.json 2> gpurun_out/ab_new$i.log; echo "new$i rc=$?"
done
timeout 900 python scripts/sweep_env.py 'KVTC_WIDE_DEFER=1' 'KVTC_CORUN_DEFLATE=1' 'KVTC_C_DEFLATE_SIDE=0' > gpurun_out/sweep_r02u.log 2>&1; echo "sweep rc=$?"
(cd _ab/old && timeout 900 python scripts/sweep_env.py 'KVTC_CORUN_DEFLATE=1' 'KVTC_C_DEFLATE_SIDE=0' > $R/gpurun_out/sweep_r02u_old.log 2>&1); echo "sweep old rc=$?"
for f in gpurun_out/ab_*.json; do python - "$f" <<'EOF'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
s = d.get("stages", {})
print(sys.argv[1], round(d["value"], 1), round(d["ms_per_step"], 2), d["clocks"]["sm_mhz"],
      {k: round(v["ms_per_step"], 2) for k, v in s.items()})
EOF
done
grep "\[sweep\]" gpurun_out/sweep_r02u.log gpurun_out/sweep_r02u_old.log
