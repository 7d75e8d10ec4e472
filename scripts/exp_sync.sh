python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_exp3.log 2>&1 || exit 1
timeout 900 python scripts/sweep_env.py KVTC_TILE_SYNC=2 KVTC_TILE_SYNC=4 KVTC_TILE_SYNC=6 KVTC_TILE_SYNC=6,KVTC_GROUP_M_QUANT=8 --iters 10 > gpurun_out/sweep_exp3.log 2>&1; echo sweep rc=$?
grep sweep gpurun_out/sweep_exp3.log
for V in 0 6; do
KVTC_TILE_SYNC=$V timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second -k "regex:gemm_kernel<[12]" --profile-from-start off --clock-control none --csv --log-file gpurun_out/ncu_exp3_$V.csv python scripts/profile_run.py > /dev/null 2>&1
python - <<PY
import csv
rows=list(csv.reader(open("gpurun_out/ncu_exp3_$V.csv")))
hdr=None; d={}
for r in rows:
    if r and r[0]=="ID": hdr=r; continue
    if hdr and len(r)==len(hdr):
        x=dict(zip(hdr,r)); d.setdefault(x["ID"],{"k":x["Kernel Name"][:22]})[x["Metric Name"]]=x["Metric Value"]
for i,x in d.items(): print("sync=$V", x["k"], {k.split("__")[1][:20]:v for k,v in x.items() if k!="k"})
PY
done
timeout 300 python scripts/cublas_ref.py 2>&1 | grep cublas
