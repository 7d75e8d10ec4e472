#!/bin/bash
# usage: scripts/codec_check.sh TAG [pytest files...]
# Codec-kernel iteration: build, GPU tests, one bench line, ncu --set full of the
# codec kernels (inflate, dequant, DEFLATE encoder) with per-line stall hotlines.
TAG=$1; shift
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1 || { tail -30 gpurun_out/build_$TAG.log; exit 1; }
if [ $# -gt 0 ]; then timeout 1200 python -m pytest "$@" -x -q > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_$TAG.log; fi
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.log; echo "bench rc=$?"
python - gpurun_out/bench_$TAG.json <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
st = d.get("stages", {})
print(sys.argv[1], round(d.get("value"), 2), round(d.get("ms_per_step"), 3), (d.get("clocks") or {}).get("sm_mhz"), round((d.get("config") or {}).get("cr"), 3),
      {k: round(v.get("ms_per_step", 0), 3) for k, v in st.items() if k.startswith("d.") or k in ("c.deflate", "c.project_quant_gemm")})
PY
timeout 600 python scripts/profile_run.py > gpurun_out/prof_${TAG}_plain.log 2>&1; echo "plain rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k "regex:inflate_fast|inflate_dequant|dequant_rows|deflate_encode" -o gpurun_out/prof_$TAG -f python scripts/profile_run.py > gpurun_out/full_$TAG.log 2>&1; echo "full rc=$?"
python scripts/ncu_hotlines.py gpurun_out/prof_$TAG.ncu-rep "inflate_fast|inflate_dequant" 30 0 > gpurun_out/hot_${TAG}_inflate.txt 2>&1
python scripts/ncu_hotlines.py gpurun_out/prof_$TAG.ncu-rep dequant_rows 30 0 > gpurun_out/hot_${TAG}_dq.txt 2>&1
python scripts/ncu_hotlines.py gpurun_out/prof_$TAG.ncu-rep deflate_encode 30 1 > gpurun_out/hot_${TAG}_deflate.txt 2>&1
ncu -i gpurun_out/prof_$TAG.ncu-rep --page details --csv > gpurun_out/details_$TAG.csv 2>&1
ncu -i gpurun_out/prof_$TAG.ncu-rep --page raw --csv > gpurun_out/raw_$TAG.csv 2>&1
rm -f gpurun_out/prof_$TAG.ncu-rep
python - gpurun_out/details_$TAG.csv <<'PY'
import csv, sys
for r in csv.DictReader(open(sys.argv[1])):
    if r['Metric Name'] in ('Duration', 'Issue Slots Busy', 'Memory Throughput', 'DRAM Throughput', 'Achieved Occupancy') :
        print(r['ID'], r['Kernel Name'][:22], r['Grid Size'], r['Metric Name'], r['Metric Value'], r['Metric Unit'])
PY
