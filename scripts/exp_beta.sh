python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_beta.log 2>&1 || exit 1
for B in 1.0 2.5; do
timeout 900 python bench.py --beta $B --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_beta$B.json 2> gpurun_out/bench_beta$B.log; echo "beta $B rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/bench_beta$B.json')); print('beta $B', round(d['value'],1), 'GB/s r_eff', d['config']['r_eff'], 'r_nz', d['config']['r_nz'], 'cr', round(d['config']['cr'],2), 'clk', d['clocks']['sm_mhz'], 'gemm frac', round(d['roofline']['frac'],3))"
done
