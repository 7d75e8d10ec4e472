#!/bin/bash
# rANS back-end tests + bench line; A/B of the wide-group epilogue fixup vs the deferred SIMT pass.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02m.log 2>&1 || { tail -30 gpurun_out/build_r02m.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_rans.py tests/test_gpu_codec.py -m gpu -x -q -s -k "rans" > gpurun_out/pytest_r02m.log 2>&1; echo "tests rc=$?"; tail -4 gpurun_out/pytest_r02m.log; grep "\[rans\]" gpurun_out/pytest_r02m.log
timeout 900 python scripts/sweep_env.py --iters 8 KVTC_WIDE_DEFER=1 > gpurun_out/sweep_r02m.log 2>&1; echo "sweep rc=$?"; grep sweep gpurun_out/sweep_r02m.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --coder rans > gpurun_out/bench_r02m_rans.json 2> gpurun_out/bench_r02m_rans.log; echo "bench rans rc=$?"; tail -3 gpurun_out/bench_r02m_rans.log
