"""Seeded synthetic inputs shared by tests, smoke() and bench.py.

This package holds NONE of the codec's arithmetic (no PCA, quantisation,
packing, DEFLATE, un-RoPE).  It plays the role of the language model that
produced the KV cache: low-rank cross-head/cross-layer structure, unequal
channel magnitudes, a non-zero mean, sink outliers and RoPE on keys, as
described in DESIGN.md §5 (recipe) — and the random sample positions the
calibration step draws, which are passed to both sides as inputs.
"""
from .synth import (DP_CASES, SHAPES, SynthSpec, dp_coefficients, generate, lengths_for, make_spec,
                    sample_positions)

__all__ = ["SynthSpec", "SHAPES", "make_spec", "generate", "sample_positions", "lengths_for", "DP_CASES",
           "dp_coefficients"]
