#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02t.log 2>&1 || { tail -30 gpurun_out/build_r02t.log; exit 1; }
timeout 300 python scripts/rans_probe.py 2>&1 | grep rans
timeout 600 ncu --set full --import-source on --clock-control none -k "regex:rans_encode|rans_decode|rans_hist|rans_copy" -c 4 -o gpurun_out/prof_r02t -f python scripts/rans_probe.py > gpurun_out/full_r02t.log 2>&1; echo "ncu rc=$?"
for k in rans_hist rans_encode rans_copy rans_decode; do echo "== $k"; ncu -i gpurun_out/prof_r02t.ncu-rep --page details -k "regex:$k" 2>/dev/null | grep -E "Duration|Issue Slots Busy|Achieved Occupancy|L1/TEX Hit|L2 Hit|Eligible Warps"; python scripts/ncu_hotlines.py gpurun_out/prof_r02t.ncu-rep "$k" 12 0; done > gpurun_out/hotlines_r02t.txt 2>&1
rm -f gpurun_out/prof_r02t.ncu-rep
