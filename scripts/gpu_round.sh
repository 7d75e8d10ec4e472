#!/bin/bash
# One GPU session: parity tests, bench line, ncu launch list + full capture of the hot kernels.
# usage: scripts/gpu_round.sh TAG [what...]   (what: tests smoke bench launches full)
# Summaries are produced on the box (gpurun_out/ comes back only if < 64 MiB).
TAG=${1:-r01}; shift
WHAT=${@:-tests bench launches full}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1 || { tail -30 gpurun_out/build_$TAG.log; exit 1; }
for w in $WHAT; do
case $w in
tests)
  timeout 1500 python -m pytest tests -m gpu -x -q -rs > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu_$TAG.log;;
smoke)
  timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/smoke_$TAG.log;;
bench)
  timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.log; echo "bench rc=$?"; python - <<PY
import json
d = json.load(open("gpurun_out/bench_$TAG.json"))
print("value", round(d["value"], 2), "ms", round(d["ms_per_step"], 2), "clocks", d["clocks"], "e2e", round(d["e2e"]["value"], 2) if d.get("e2e") else None)
print("roofline", {k: d["roofline"][k] for k in ("achieved", "frac", "traffic")})
for k, v in d["stages"].items(): print("  ", k, {a: round(b, 3) for a, b in v.items()})
PY
  ;;
launches)
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_$TAG.csv python scripts/profile_run.py > gpurun_out/launches_$TAG.log 2>&1; echo "launches rc=$?";;
full)
  timeout 1500 ncu --set full --clock-control none --import-source on --profile-from-start off -k "regex:gemm_kernel|deflate_encode|inflate_fast|gather_kernel|dequant_kernel" -o gpurun_out/prof_$TAG -f python scripts/profile_run.py > gpurun_out/full_$TAG.log 2>&1; echo "full rc=$?"
  python scripts/ncu_summary.py gpurun_out/launches_$TAG.csv gpurun_out/prof_$TAG.ncu-rep gpurun_out/summary_$TAG.md gpurun_out/traffic_$TAG.json "$TAG" > /dev/null 2>&1
  for k in "gemm_kernel<1" "gemm_kernel<2" deflate_encode inflate_fast gather_kernel dequant_kernel; do echo "== $k"; python scripts/ncu_hotlines.py gpurun_out/prof_$TAG.ncu-rep "$k" 20; done > gpurun_out/hotlines_$TAG.txt 2>&1
  ls -la gpurun_out/prof_$TAG.ncu-rep
  if [ $(stat -c %s gpurun_out/prof_$TAG.ncu-rep) -gt 50000000 ]; then rm gpurun_out/prof_$TAG.ncu-rep; echo "report too large, removed"; fi;;
esac
done
