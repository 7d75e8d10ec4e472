#!/bin/bash
# Schedule knobs re-measured with the faster codec kernels.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02q.log 2>&1 || { tail -30 gpurun_out/build_r02q.log; exit 1; }
timeout 1500 python scripts/sweep_env.py --iters 12 KVTC_D_INFLATE_SIDE=1 KVTC_D_INFLATE_SIDE=1,KVTC_CORUN_INFLATE=2 KVTC_D_INFLATE_SIDE=1,KVTC_CORUN_INFLATE=8 > gpurun_out/sweep_r02q.log 2>&1; echo "sweep rc=$?"; grep sweep gpurun_out/sweep_r02q.log | cut -c1-100
