#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02r.log 2>&1 || { tail -30 gpurun_out/build_r02r.log; exit 1; }
timeout 600 ncu --set full --import-source on --clock-control none --profile-from-start off -k "regex:inflate_fast|deflate_encode" -c 3 -o gpurun_out/prof_r02r -f python scripts/profile_run.py > gpurun_out/full_r02r.log 2>&1; echo "ncu rc=$?"
python scripts/ncu_hotlines.py gpurun_out/prof_r02r.ncu-rep "inflate_fast" 30 0 > gpurun_out/hotlines_r02r.txt 2>&1
python scripts/ncu_hotlines.py gpurun_out/prof_r02r.ncu-rep "deflate_encode" 30 1 >> gpurun_out/hotlines_r02r.txt 2>&1
ncu -i gpurun_out/prof_r02r.ncu-rep --page details --launch-skip 2 --launch-count 1 2>/dev/null | grep -E "Duration|Registers|Achieved Occupancy|Theoretical Occupancy|Block Limit|Waves|Issue Slots" >> gpurun_out/hotlines_r02r.txt
rm -f gpurun_out/prof_r02r.ncu-rep
