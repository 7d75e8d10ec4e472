#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02s.log 2>&1 || { tail -30 gpurun_out/build_r02s.log; exit 1; }
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -k "regex:gemm_kernel" -c 1 -o gpurun_out/prof_r02s -f python scripts/profile_run.py > gpurun_out/full_r02s.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/prof_r02s.ncu-rep --page source --csv --print-source sass > gpurun_out/sass_r02s.csv 2>/dev/null
ncu -i gpurun_out/prof_r02s.ncu-rep --page details 2>/dev/null | grep -E "Duration|Tensor|Issue Slots|Eligible|DRAM Through|L2 Hit|L1/TEX Hit|Registers|Stall" > gpurun_out/details_r02s.txt
rm -f gpurun_out/prof_r02s.ncu-rep
