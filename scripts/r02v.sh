#!/bin/bash
# wide-group fixup with batched loads: parity, isolated GEMM time (launch list), bench A/B vs e0b4133
mkdir -p gpurun_out
R=$PWD
timeout 900 python -m pytest tests/test_gpu_stages.py tests/test_gpu_codec.py -m gpu -x -q 2>&1 | tail -3
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_r02v.csv python scripts/profile_run.py > gpurun_out/launches_r02v.log 2>&1; echo "launches rc=$?"
grep gemm_kernel gpurun_out/launches_r02v.csv | awk -F'","' '{print $5, $(NF)}' | head -8
for i in 1 2; do
  timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/ab_v_new$i.json 2> gpurun_out/ab_v_new$i.log; echo "new$i rc=$?"
  (cd _ab/old && timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu > $R/gpurun_out/ab_v_old$i.json 2> $R/gpurun_out/ab_v_old$i.log); echo "old$i rc=$?"
done
timeout 900 python scripts/sweep_env.py 'KVTC_WIDE_DEFER=1' 'KVTC_C_DEFLATE_SIDE=0' > gpurun_out/sweep_r02v.log 2>&1; echo "sweep rc=$?"
for f in gpurun_out/ab_v_*.json; do python - "$f" <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
s = d.get("stages", {})
print(sys.argv[1], round(d["value"], 1), round(d["ms_per_step"], 2), d["clocks"]["sm_mhz"],
      {k: round(v["ms_per_step"], 2) for k, v in s.items()})
PY
done
grep "\[sweep\]" gpurun_out/sweep_r02v.log
