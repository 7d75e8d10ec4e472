#!/bin/bash
# Raster group sweep of the codec GEMMs (DRAM traffic vs time under the power cap) + accumulation emulation.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02p.log 2>&1 || { tail -30 gpurun_out/build_r02p.log; exit 1; }
timeout 1200 python scripts/sweep_env.py --iters 8 KVTC_GROUP_M_QUANT=8 KVTC_GROUP_M_QUANT=4 KVTC_GROUP_M_QUANT=32 KVTC_GROUP_M_RECON=8 KVTC_GROUP_M_RECON=32 > gpurun_out/sweep_r02p.log 2>&1; echo "sweep rc=$?"; grep sweep gpurun_out/sweep_r02p.log | cut -c1-200
for gm in 8 16 32; do
KVTC_GROUP_M_QUANT=$gm timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off -k "regex:gemm_kernel" -c 2 --csv python scripts/profile_run.py 2>/dev/null | grep -E "dram__bytes_read|gpu__time" | cut -c1-220 > gpurun_out/dram_gm$gm.csv; echo "gm $gm"; cat gpurun_out/dram_gm$gm.csv | awk -F'","' '{print $(NF-2), $NF}'
done
timeout 1200 python scripts/accum_emulation.py > gpurun_out/accum_r02p.log 2>&1; echo "accum rc=$?"; tail -5 gpurun_out/accum_r02p.log
