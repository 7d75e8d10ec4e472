python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_exp18.log 2>&1 || exit 1
for V in "KVTC_NO_DIRECT=0" "KVTC_NO_DIRECT=1"; do
env $V timeout 900 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second,dram__bytes_read.sum,lts__t_sector_hit_rate.pct -k regex:gemm --profile-from-start off --clock-control none -c 2 --csv --log-file gpurun_out/ncu_exp18.csv python scripts/profile_run.py > /dev/null 2>&1
python - "$V" <<'PY'
import csv, sys
rows=list(csv.reader(open("gpurun_out/ncu_exp18.csv")))
hdr=None; d={}
for r in rows:
    if r and r[0]=="ID": hdr=r; continue
    if hdr and len(r)==len(hdr):
        x=dict(zip(hdr,r)); d.setdefault(x["ID"],{"k":x["Kernel Name"][:20]})[x["Metric Name"]]=x["Metric Value"]
for i,x in list(d.items())[:2]: print(sys.argv[1], x["k"], {k.split("__")[1][:22]:v for k,v in x.items() if k!="k"})
PY
done
