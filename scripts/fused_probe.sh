#!/bin/bash
# Reconstruction GEMM alone on the bench shape: fused dequantising producer vs D^ through TMA (measurement).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_probe.log 2>&1 || { tail -30 gpurun_out/build_probe.log; exit 1; }
timeout 600 python scripts/fused_probe.py "$@" > gpurun_out/probe.log 2>&1; echo "probe rc=$?"; grep probe gpurun_out/probe.log
