"""Joint cross-shard compression of a layer-sharded cache.

P:L386-387 (Table 3 caption): with the model split across GPUs (pipeline
parallel), KVTC is applied to each GPU's chunk of the cache separately (P:L443,
`bench.py --config llama70b_shard`), but "these chunks could be compressed
jointly for higher accuracy".  Reading Q23: one basis (mu, V)
and one plan over the concatenated features of all shards (p = sum p_g, layers
in shard order).  Rank g holds the rows X_g of its layers and the rows V_g of V
for its features, so

    D = X V - mu V = sum_g X_g V_g - mu V                       (block identity)

compress  : rank g projects its partial P_g = X_g V_g (tcgen05 GEMM,
            kvtc_stage_project_partial; rank 0 also subtracts mu V), the partials
            are summed by a reduce-scatter over token rows (NCCL; tile-aligned
            slices of 128 tokens), and rank r quantises + packs + DEFLATEs its
            slice with the shared plan: together the ranks hold exactly the
            single-device payload of the joint features (up to the fp32
            summation order of the partials);
decompress: rank r inflates + dequantises its slice (D^ rows, fp16), an
            all-gather gives every rank all rows of D^, and rank g rebuilds only
            its own layers X^_g = D^ V_{d,g}^T + mu_g (the layer-range
            reconstruction of kvtc_stage_reconstruct).
The exchanged bytes are fp32 partials (m x r_nz x 4 B) on compress and fp16 D^
(m x r_nz x 2 B) on decompress.  Every arithmetic step runs in libkvtc.so; this
module is argument marshalling plus the two collectives (torch.distributed:
NCCL on GPUs, gloo in the CPU tests).
"""
from __future__ import annotations

import torch

TILE = 128


def row_partition(m: int, world: int):
    """Tile-aligned token slices: rank r owns rows [r0, r1) of the m middle
    tokens; every rank's slice is `per` tiles long in the padded exchange buffer
    of world * per * 128 rows.  Returns (per_rows, [(r0, r1) per rank])."""
    tiles = (m + TILE - 1) // TILE
    per = (tiles + world - 1) // world if world else 0
    out = []
    for r in range(world):
        r0 = min(m, r * per * TILE)
        r1 = min(m, (r + 1) * per * TILE)
        out.append((r0, r1))
    return per * TILE, out


def reduce_scatter_rows(P: torch.Tensor, world: int, rank: int, group=None) -> torch.Tensor:
    """Sum [m x c] partials over the ranks and return this rank's tile-aligned row
    slice (reduce-scatter; gloo lacks it, so there the sum is an all-reduce and
    the slice is taken locally)."""
    import torch.distributed as dist
    m, c = P.shape
    per, parts = row_partition(m, world)
    r0, r1 = parts[rank]
    if world == 1:
        return P[r0:r1].contiguous()
    buf = torch.zeros(world * per, c, dtype=P.dtype, device=P.device)
    buf[:m] = P
    if dist.get_backend(group) == "nccl":
        out = torch.empty(per, c, dtype=P.dtype, device=P.device)
        dist.reduce_scatter_tensor(out, buf, group=group)
    else:
        dist.all_reduce(buf, group=group)
        out = buf[rank * per:(rank + 1) * per]
    return out[:r1 - r0].contiguous()


def all_gather_rows(D: torch.Tensor, m: int, world: int, rank: int, group=None) -> torch.Tensor:
    """The inverse exchange: every rank's row slice -> all m rows on every rank."""
    import torch.distributed as dist
    per, parts = row_partition(m, world)
    if world == 1:
        return D.contiguous()
    c = D.shape[1]
    mine = torch.zeros(per, c, dtype=D.dtype, device=D.device)
    mine[:D.shape[0]] = D
    full = torch.empty(world * per, c, dtype=D.dtype, device=D.device)
    dist.all_gather_into_tensor(full, mine, group=group)
    return full[:m].contiguous()


class JointShard:
    """One rank's side of the joint codec for one stream (keys or values).

    basis / plan: the joint basis and plan (kvtc.Basis / kvtc.Plan over all
    layers, identical on every rank); layer_begin / layer_end: this rank's layers
    of the joint feature order."""

    def __init__(self, K, basis, plan, layer_begin: int, layer_end: int, group=None):
        import torch.distributed as dist
        self.K, self.basis, self.plan = K, basis, plan
        self.lb, self.le = layer_begin, layer_end
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        L, h, d = basis.shape
        self.hd = h * d
        self.L = L

    def partial(self, view, sinks: int, m: int, unrope: bool, inv_freq=None, pairing: int = 0, add_bias=None):
        """This shard's partial projection P_g [m x r_nz] fp32 (view: the shard's
        own layers, shape (le - lb, h, d))."""
        K = self.K
        X = K.gather(view, sinks, m, unrope, inv_freq, pairing)
        bias = (self.rank == 0) if add_bias is None else add_bias
        return K.project_partial(self.basis, self.plan, X, self.lb * self.hd, self.le * self.hd, bias)

    def compress(self, view, sinks: int, window: int, unrope: bool, inv_freq=None, pairing: int = 0,
                 chunk_bytes: int = 65536):
        """-> (payload of this rank's rows, its DEFLATE section, (r0, r1), m)."""
        K = self.K
        m = max(0, view.tokens - sinks - window)
        P = self.partial(view, sinks, m, unrope, inv_freq, pairing)
        D = reduce_scatter_rows(P, self.world, self.rank, self.group)
        _, parts = row_partition(m, self.world)
        payload = K.quantize_pack(self.plan, D) if D.shape[0] else torch.zeros(0, dtype=torch.uint8, device="cuda")
        section = K.deflate(payload, chunk_bytes) if payload.numel() else None
        return payload, section, parts[self.rank], m

    def decompress(self, section, rows: int, m: int, sinks: int, out_layers, pos0: int = 0):
        """Inflate + dequantise this rank's rows, all-gather D^, rebuild this shard's
        layers into out_layers (list of the shard's per-layer [tokens, h, d] bf16
        tensors, rows sinks .. sinks + m are written)."""
        K = self.K
        ncols = sum(z for (_, z, _) in self.plan.info().groups)
        ld = max(8, (ncols + 7) // 8 * 8)
        if rows:
            payload = K.inflate(section, self.plan.payload_bytes(rows))
            Dh = K.dequantize(self.plan, payload, rows, ld)
        else:
            Dh = torch.zeros(0, ld, dtype=torch.float16, device="cuda")
        Dall = all_gather_rows(Dh, m, self.world, self.rank, self.group)
        # a view of the joint layer count whose non-owned layers are never written
        tokens = out_layers[0].shape[0]
        dummy = out_layers[0]
        layers = [out_layers[l - self.lb] if self.lb <= l < self.le else dummy for l in range(self.L)]
        view = K.KVView(layers, pos0=pos0, tokens=tokens)
        K.reconstruct(self.basis, self.plan, Dall, m, sinks, self.lb, self.le, view)
        return Dall
