cat > /tmp/cb.py <<'PY'
import torch
for (M,N,K) in [(32636,4352,32768),(32636,32768,4352)]:
    a = torch.randn(M, K, device="cuda", dtype=torch.bfloat16); b = torch.randn(K, N, device="cuda", dtype=torch.bfloat16)
    for _ in range(2): c = a @ b
    torch.cuda.synchronize()
PY
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second,launch__grid_size,launch__block_size,launch__cluster_dim_x,launch__cluster_dim_y,launch__shared_mem_per_block_dynamic,lts__t_bytes.sum --clock-control none --csv python /tmp/cb.py 2>&1 | grep -v "^==" | cut -c1-400 > gpurun_out/cublas_ncu.csv
cat gpurun_out/cublas_ncu.csv | python -c "
import csv,sys
rows=list(csv.reader(sys.stdin))
h=rows[0]
for r in rows[1:]:
    d=dict(zip(h,r)); print(d.get('Kernel Name','')[:150], d.get('Metric Name'), d.get('Metric Value'))
"
