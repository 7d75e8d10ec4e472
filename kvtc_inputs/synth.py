"""Synthetic KV caches shaped like the paper's models.

Per (shape, stream) a fixed "model" is drawn once from the seed:
  * G in R^{K x p}, entries N(0, 1/p) — K latent directions shared by every
    layer and head (the cross-head / cross-layer low-rank structure of P:L101-111);
  * spectrum lambda_i = c * (1 + i/16)^(-beta), c set so the per-feature RMS of
    the low-rank part is rho*sqrt(0.99) (unequal channel magnitudes);
  * mean mu_f ~ N(0, mu_sd^2) (keys 0.5, values 0.05; our choice — the paper only
    implies a non-zero mean by centring).
Rows of a conversation: x_t = mu + s_t * (sum_i sqrt(lambda_i) z_{t,i} G_i + n_t),
z, n ~ N(0, 1) (noise n at 1 % of the variance), s_t = 8 for absolute positions
< 4 (sink outliers), else 1.  Keys are then rotated by RoPE
(HF convention, fp32, half-split pairing) at their absolute positions, as the
model would have done before caching them; values are not.
Everything is rounded once to bf16.  Layout [layers, tokens, kv_heads, head_dim].
"""
from __future__ import annotations

import math
from dataclasses import dataclass, replace

import numpy as np
import torch

BASE_SEED = 0x4B565443


def _splitmix64(x: int) -> int:
    x = (x + 0x9E3779B97F4A7C15) & 0xFFFFFFFFFFFFFFFF
    z = x
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & 0xFFFFFFFFFFFFFFFF
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & 0xFFFFFFFFFFFFFFFF
    return z ^ (z >> 31)


def _fnv1a(s: str) -> int:
    h = 0xCBF29CE484222325
    for ch in s.encode():
        h = ((h ^ ch) * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return h


def seed_for(config: str, stream: int, conversation: int) -> int:
    x = BASE_SEED ^ _splitmix64(_fnv1a(config))
    x = _splitmix64(x ^ (stream + 1) * 0x9E37)
    x = _splitmix64(x ^ (conversation + 7) * 0x85EB)
    return x & 0x7FFFFFFFFFFFFFFF


@dataclass(frozen=True)
class SynthSpec:
    name: str
    layers: int
    kv_heads: int
    head_dim: int
    latent: int               # K
    beta: float = 1.5
    rope_base: float = 500000.0
    rho: tuple = (1.0, 0.35)          # (keys, values)
    mu_sd: tuple = (0.5, 0.05)
    noise_frac: float = 0.01
    sink_scale: float = 8.0
    sinks: int = 4

    @property
    def p(self) -> int:
        return self.layers * self.kv_heads * self.head_dim

    def inv_freq(self) -> torch.Tensor:
        """The model's RoPE frequencies (fp32), as HF computes them."""
        d = self.head_dim
        return 1.0 / (self.rope_base ** (torch.arange(0, d, 2, dtype=torch.int64).float() / d))


SHAPES = {
    # BASELINE.json configs[0]: 1 layer, 2 KV heads x 64, 512 tokens
    "toy": SynthSpec("toy", 1, 2, 64, latent=32, rope_base=10000.0),
    # configs[1]: Llama-3.1-8B shape (32 x 8 x 128), public rope_theta 5e5.  Latent rank
    # p/8 and 0.1 % noise: frozen after the tuning run of DESIGN.md §5 (r_eff at CR 16 ~ 4.3K)
    "llama8b": SynthSpec("llama8b", 32, 8, 128, latent=4096, rope_base=500000.0, noise_frac=0.001),
    # configs[2]: Mistral-NeMo-12B shape (40 x 8 x 128), rope_theta 1e6
    "nemo12b": SynthSpec("nemo12b", 40, 8, 128, latent=5120, rope_base=1000000.0, noise_frac=0.001),
    # configs[3]: Llama-3.3-70B, one 10-layer shard of 80 x 8 x 128
    "llama70b_shard": SynthSpec("llama70b_shard", 10, 8, 128, latent=1280, rope_base=500000.0, noise_frac=0.001),
}


def make_spec(base: str, **over) -> SynthSpec:
    """A named shape, optionally with fields overridden (e.g. name=..., layers=...)."""
    return replace(SHAPES[base], **over) if over else SHAPES[base]


_MODEL_CACHE: dict = {}


def _model(spec: SynthSpec, stream: int, device):
    key = (spec, stream, str(device))
    if key in _MODEL_CACHE:
        return _MODEL_CACHE[key]
    g = torch.Generator(device="cpu").manual_seed(seed_for(spec.name, stream, -1))
    p, K = spec.p, spec.latent
    rho = spec.rho[stream]
    lam = (1.0 + torch.arange(K, dtype=torch.float64) / 16.0) ** (-spec.beta)
    lam = lam * (p * rho * rho * (1.0 - spec.noise_frac) / lam.sum())
    mu = torch.randn(p, generator=g, dtype=torch.float32) * spec.mu_sd[stream]
    # G is drawn on the target device in row blocks from a device generator
    gd = torch.Generator(device=device).manual_seed(seed_for(spec.name, stream, -2))
    G = torch.randn(K, p, generator=gd, device=device, dtype=torch.float32) / math.sqrt(p)
    G.mul_(lam.sqrt().to(device=device, dtype=torch.float32)[:, None])
    out = (mu.to(device), G, rho * math.sqrt(spec.noise_frac))
    if len(_MODEL_CACHE) > 8:
        _MODEL_CACHE.clear()
    _MODEL_CACHE[key] = out
    return out


def _rope_hf(x: torch.Tensor, pos: torch.Tensor, inv_freq: torch.Tensor) -> torch.Tensor:
    """HF rotary embedding, half-split: x*cos + rotate_half(x)*sin (fp32)."""
    freqs = pos.float()[:, None] * inv_freq.to(x.device)[None, :]
    emb = torch.cat([freqs, freqs], dim=-1)
    cos, sin = emb.cos()[:, None, :], emb.sin()[:, None, :]
    h = x.shape[-1] // 2
    rot = torch.cat([-x[..., h:], x[..., :h]], dim=-1)
    return x * cos + rot * sin


@torch.no_grad()
def generate(spec: SynthSpec, stream: int, tokens: int, pos0: int = 0, conversation: int = 0,
             device="cpu", chunk: int = 4096, out: torch.Tensor | None = None) -> torch.Tensor:
    """bf16 [layers, tokens, kv_heads, head_dim] for stream 0 (keys) / 1 (values)."""
    device = torch.device(device)
    mu, G, noise_sd = _model(spec, stream, device)
    l, h, d = spec.layers, spec.kv_heads, spec.head_dim
    if out is None:
        out = torch.empty(l, tokens, h, d, dtype=torch.bfloat16, device=device)
    gen = torch.Generator(device=device).manual_seed(seed_for(spec.name, stream, conversation))
    invf = spec.inv_freq()
    for t0 in range(0, tokens, chunk):
        t1 = min(tokens, t0 + chunk)
        n = t1 - t0
        z = torch.randn(n, spec.latent, generator=gen, device=device, dtype=torch.float32)
        x = z @ G
        x += torch.randn(n, spec.p, generator=gen, device=device, dtype=torch.float32) * noise_sd
        pos = torch.arange(pos0 + t0, pos0 + t1, device=device)
        sink = (pos < spec.sinks).float() * (spec.sink_scale - 1.0) + 1.0
        x *= sink[:, None]
        x += mu[None, :]
        x = x.view(n, l, h, d)
        if stream == 0:
            x = _rope_hf(x.reshape(n, l * h, d), pos, invf).view(n, l, h, d)
        out[:, t0:t1] = x.permute(1, 0, 2, 3).to(torch.bfloat16)
    return out


def lengths_for(n_conv: int, lo: int, hi: int, seed: int = 0) -> list:
    """Conversation lengths t_c ~ UniformInt[lo, hi] (multi-conversation config)."""
    rng = np.random.default_rng(seed)
    return [int(x) for x in rng.integers(lo, hi + 1, size=n_conv)]


def sample_positions(lengths, n: int, sinks: int = 4, seed: int = 0) -> np.ndarray:
    """The calibration draw: n positions without replacement from the
    pooled positions of all sequences, excluding sinks.  [n, 2] int64 of
    (sequence, token index), in draw order."""
    pool = []
    for si, t in enumerate(lengths):
        tok = np.arange(sinks, t, dtype=np.int64)
        pool.append(np.stack([np.full_like(tok, si), tok], axis=1))
    pool = np.concatenate(pool, axis=0)
    if n > len(pool):
        raise ValueError("n exceeds the pool of non-sink positions")
    rng = np.random.default_rng(seed)
    idx = rng.choice(len(pool), size=n, replace=False)
    return pool[idx]


# DP-parity inputs at production shape (tests/test_gpu_calib_dp.py,
# scripts/make_dp_golden.py): projected calibration coefficients P [n x r] whose
# column scales mimic a PCA spectrum.  kind "decay": scale_i = 3 (1 + i)^-0.8
# plus a per-column offset (as the small DP cases); kind "flat_tail": a head of
# `head` PCs decaying as 3 / (1 + i) and a flat noise floor `tail` after it, so
# the optimum spends the leftover budget on 256- / 1024-PC int groups.  fp32.
DP_CASES = {
    "decay_b32768": dict(kind="decay", n=128, r=2200, budget=32768, seed=7),
    "tail_1024": dict(kind="flat_tail", n=64, r=2300, budget=8000, head=200, tail=0.02, seed=1),
    "tail_256": dict(kind="flat_tail", n=64, r=2300, budget=6000, head=128, tail=0.01, seed=4),
}


def dp_coefficients(kind: str, n: int, r: int, seed: int, head: int = 0, tail: float = 0.0, **_) -> np.ndarray:
    rng = np.random.default_rng(seed)
    i = np.arange(r)
    if kind == "decay":
        scale = (1.0 + i) ** -0.8 * 3.0
        P = rng.standard_normal((n, r)) * scale + rng.normal(0, 0.3, (1, r))
    elif kind == "flat_tail":
        scale = np.where(i < head, 3.0 * (1.0 + i) ** -1.0, tail)
        P = rng.standard_normal((n, r)) * scale
    else:
        raise KeyError(kind)
    return P.astype(np.float32)
