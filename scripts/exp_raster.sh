python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_exp1.log 2>&1 || exit 1
V="KVTC_GROUP_M_QUANT=1 KVTC_GROUP_M_QUANT=2 KVTC_GROUP_M_QUANT=8 KVTC_GROUP_M_QUANT=17 KVTC_GROUP_M_QUANT=37 KVTC_HINT_B=2 KVTC_HINT_A=1 KVTC_HINT_A=1,KVTC_HINT_B=2 KVTC_GROUP_M_RECON=4 KVTC_GROUP_M_RECON=8 KVTC_GROUP_M_RECON=37 KVTC_GROUP_M_RECON=64"
timeout 900 python scripts/sweep_env.py $V --iters 5 > gpurun_out/sweep_exp1.log 2>&1; echo sweep rc=$?
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second -k regex:gemm_kernel --clock-control none --csv --log-file gpurun_out/ncu_exp1.csv python scripts/sweep_env.py $V --iters 1 > gpurun_out/ncu_exp1.log 2>&1; echo ncu rc=$?
grep sweep gpurun_out/sweep_exp1.log
