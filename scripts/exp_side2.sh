python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_exp23.log 2>&1 || exit 1
timeout 1500 python scripts/sweep_env.py KVTC_C_DEFLATE_SIDE=0 KVTC_C_DEFLATE_SIDE=0 KVTC_C_DEFLATE_SIDE=0,KVTC_C_GATHER_SIDE=0 KVTC_C_DEFLATE_SIDE=0 --iters 10 > gpurun_out/sweep_exp23.log 2>&1; echo sweep rc=$?
grep sweep gpurun_out/sweep_exp23.log | cut -c1-140
