python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_exp9.log 2>&1 || exit 1
./scripts/probe/cluster_occ
timeout 1200 python scripts/sweep_env.py KVTC_NO_DIRECT=1 KVTC_GROUP_M_QUANT=2 KVTC_GROUP_M_QUANT=8 KVTC_GROUP_M_RECON=8 KVTC_GROUP_M_RECON=32 --iters 10 > gpurun_out/sweep_exp9.log 2>&1; echo sweep rc=$?
grep sweep gpurun_out/sweep_exp9.log | cut -c1-330
