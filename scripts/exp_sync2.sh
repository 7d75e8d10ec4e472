python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_exp21.log 2>&1 || exit 1
timeout 1500 python scripts/sweep_env.py KVTC_TILE_SYNC=0 KVTC_TILE_SYNC=2 KVTC_GROUP_M_QUANT=8 KVTC_GROUP_M_RECON=8 KVTC_GROUP_M_QUANT=32 --iters 10 > gpurun_out/sweep_exp21.log 2>&1; echo sweep rc=$?
grep sweep gpurun_out/sweep_exp21.log | cut -c1-120
