#!/bin/bash
# ncu --set full of the rewritten inflater and dequantiser (default encoder limit 15) + stage tests.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_z.log 2>&1 || { tail -30 gpurun_out/build_z.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_stages.py -x -q > gpurun_out/pytest_z.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_z.log
timeout 600 python scripts/profile_run.py > gpurun_out/prof_z_plain.log 2>&1; echo "plain rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k "regex:inflate_fast|dequant_rows" -o gpurun_out/prof_z -f python scripts/profile_run.py > gpurun_out/full_z.log 2>&1; echo "full rc=$?"
python scripts/ncu_hotlines.py gpurun_out/prof_z.ncu-rep inflate_fast 40 0 > gpurun_out/hot_z_inflate.txt 2>&1
python scripts/ncu_hotlines.py gpurun_out/prof_z.ncu-rep dequant_rows 40 0 > gpurun_out/hot_z_dq0.txt 2>&1
python scripts/ncu_hotlines.py gpurun_out/prof_z.ncu-rep dequant_rows 40 1 > gpurun_out/hot_z_dq1.txt 2>&1
ncu -i gpurun_out/prof_z.ncu-rep --page details --csv > gpurun_out/details_z.csv 2>&1
ncu -i gpurun_out/prof_z.ncu-rep --page raw --csv > gpurun_out/raw_z.csv 2>&1
rm -f gpurun_out/prof_z.ncu-rep
