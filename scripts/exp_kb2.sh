python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_exp19.log 2>&1 || exit 1
KVTC_KB2=6 timeout 900 python -m pytest tests/test_gpu_stages.py tests/test_gpu_codec.py tests/test_gpu_batch.py -x -q > gpurun_out/pytest_exp19.log 2>&1; echo "pytest kb2 rc=$?"; tail -3 gpurun_out/pytest_exp19.log | cut -c1-300
timeout 1200 python scripts/sweep_env.py KVTC_KB2=2 KVTC_KB2=4 KVTC_KB2=6 --iters 10 > gpurun_out/sweep_exp19.log 2>&1; echo sweep rc=$?
grep sweep gpurun_out/sweep_exp19.log | cut -c1-200
for V in "KVTC_KB2=0" "KVTC_KB2=6"; do
env $V timeout 900 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second,dram__bytes_read.sum -k regex:gemm --profile-from-start off --clock-control none --csv --log-file gpurun_out/ncu_exp19.csv python scripts/profile_run.py > /dev/null 2>&1
python - "$V" <<'PY'
import csv, sys
rows=list(csv.reader(open("gpurun_out/ncu_exp19.csv")))
hdr=None; d={}
for r in rows:
    if r and r[0]=="ID": hdr=r; continue
    if hdr and len(r)==len(hdr):
        x=dict(zip(hdr,r)); d.setdefault(x["ID"],{"k":x["Kernel Name"][:20]})[x["Metric Name"]]=x["Metric Value"]
for i,x in list(d.items())[:4]: print(sys.argv[1], x["k"], {k.split("__")[1][:22]:v for k,v in x.items() if k!="k"})
PY
done
