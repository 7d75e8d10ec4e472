python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_exp4.log 2>&1 || exit 1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_exp4.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_exp4.log
timeout 900 python scripts/sweep_env.py KVTC_GROUP_M_QUANT=2 KVTC_GROUP_M_QUANT=8 KVTC_GROUP_M_QUANT=16 KVTC_GROUP_M_RECON=8 KVTC_GROUP_M_RECON=32 KVTC_C_GATHER_SIDE=0 KVTC_C_DEFLATE_SIDE=0 --iters 10 > gpurun_out/sweep_exp4.log 2>&1; echo sweep rc=$?
grep sweep gpurun_out/sweep_exp4.log | cut -c1-200
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_exp4.json 2> gpurun_out/bench_exp4.log; echo "bench rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/bench_exp4.json')); print(d['value'], d['ms_per_step'], d['clocks'], d['e2e'])"
