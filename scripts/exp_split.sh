python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_exp5.log 2>&1 || exit 1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_exp5.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_exp5.log
timeout 900 python scripts/sweep_env.py KVTC_C_SPLIT=0 KVTC_TILE_SYNC=2 --iters 10 > gpurun_out/sweep_exp5.log 2>&1; echo sweep rc=$?
grep sweep gpurun_out/sweep_exp5.log | cut -c1-330
for V in 0 6; do
KVTC_TILE_SYNC=$V timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second,lts__t_bytes.sum -k regex:gemm --profile-from-start off --clock-control none --csv --log-file gpurun_out/ncu_exp5_$V.csv python scripts/profile_run.py > /dev/null 2>&1
python - <<PY
import csv
rows=list(csv.reader(open("gpurun_out/ncu_exp5_$V.csv")))
hdr=None; d={}
for r in rows:
    if r and r[0]=="ID": hdr=r; continue
    if hdr and len(r)==len(hdr):
        x=dict(zip(hdr,r)); d.setdefault(x["ID"],{"k":x["Kernel Name"][:22]})[x["Metric Name"]]=x["Metric Value"]
for i,x in d.items(): print("sync=$V", x["k"], {k.split("__")[1][:24]:v for k,v in x.items() if k!="k"})
PY
done
