"""KVTC oracle — TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct CPU implementation of what the KVTC hot path
computes (arXiv 2511.01815, "KV cache Transform Coding"), written from PAPER.md
and the readings listed in DESIGN.md §3.  It is fp64 NumPy (plus one plain-C
file for the literal DP loop) and shares NO code with the CUDA product path in
``paper_2511_01815_b200/``: neither imports the other.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import anything in here.

Citation keys used in docstrings: ``P:Lnnn`` = /root/reference/PAPER.md line
nnn; ``Q<k>`` / ``R<k>`` = the reading numbered k in DESIGN.md §3.

Modules
  numerics  IEEE rounding to fp16/bf16/fp32 and OCP E4M3 (R3-R5, Q3, Q4)
  rope      un-RoPE / RoPE (Q10, R1, R7)
  quant     grouped scalar quantiser (Q1-Q5)
  dp        literal DP of P:L1541-1603, E/Z tables (Q9), brute force, backtrack
  pca       calibration: gather, mean, PCA basis
  layout    payload byte layout
  entropy   chunked raw DEFLATE through zlib (Q15)
  codec     compress / decompress / CR

Parity status per function is stated in each module header; functions with no
pin other than themselves say "parity unpinned" (also listed in DESIGN.md).
"""
