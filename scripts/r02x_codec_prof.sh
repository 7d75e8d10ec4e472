#!/bin/bash
# Codec-kernel profile: ncu --set full with source for the DEFLATE encoder, the inflater and the dequantiser.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_x.log 2>&1 || { tail -30 gpurun_out/build_x.log; exit 1; }
timeout 600 python scripts/profile_run.py > gpurun_out/prof_x_plain.log 2>&1; echo "plain rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k "regex:deflate_encode|inflate_fast|dequant_kernel" -o gpurun_out/prof_x -f python scripts/profile_run.py > gpurun_out/full_x.log 2>&1; echo "full rc=$?"
for k in inflate_fast deflate_encode dequant_kernel; do
  python scripts/ncu_hotlines.py gpurun_out/prof_x.ncu-rep $k 40 0 > gpurun_out/hot_x_$k.txt 2>&1
done
python scripts/ncu_hotlines.py gpurun_out/prof_x.ncu-rep deflate_encode 40 1 > gpurun_out/hot_x_deflate1.txt 2>&1
ncu -i gpurun_out/prof_x.ncu-rep --page details --csv > gpurun_out/details_x.csv 2>&1
ls -la gpurun_out/prof_x.ncu-rep
