#!/bin/bash
# One GPU session: parity tests, bench line, ncu launch list + full capture of the hot kernels.
# usage: scripts/gpu_round.sh TAG [what...]   (what: tests bench launches full)
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
  timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.log; echo "bench rc=$?"; cat gpurun_out/bench_$TAG.json | head -c 600; echo;;
launches)
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_$TAG.csv python scripts/profile_run.py > gpurun_out/launches_$TAG.log 2>&1; echo "launches rc=$?";;
full)
  timeout 1500 ncu --set full --clock-control none --import-source on --profile-from-start off -o gpurun_out/prof_$TAG -f python scripts/profile_run.py > gpurun_out/full_$TAG.log 2>&1; echo "full rc=$?";;
esac
done
