"""Joint cross-shard compression (reading Q23): one
basis over the features of all layer shards; each shard projects its partial
X_g V_g on the tensor cores (kvtc_stage_project_partial), the partials are
summed (the reduce-scatter's arithmetic, done here on one GPU with the shards
in turn), quantised / packed with the shared plan, and each shard rebuilds only
its own layers from the gathered D^ (paper_2511_01815_b200/joint.py).

Parity: the summed partials against the oracle's fp64 projection of the joint
features (the codes gate of DESIGN.md §7), the shard reconstruction against the
oracle's decompression of the same payload, and the paper's claim that joint
compression is more accurate than per-shard compression at equal bits."""
import numpy as np
import pytest
import torch

from oracle import layout as OL
from oracle import numerics as ON
from oracle import pca as OPCA
from oracle import quant as OQ
from oracle import rope as OR
from tests import gpu_env as E

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def K():
    from paper_2511_01815_b200 import kvtc
    kvtc.device_check()
    return kvtc


def _bf16_np(t):
    return t.float().cpu().numpy().astype(np.float64)


@pytest.mark.parametrize("tokens,pos0", [(1000, 0), (132 + 128 * 3, 77)])
def test_joint_partials_vs_oracle(K, tokens, pos0):
    from paper_2511_01815_b200.joint import JointShard
    spec, invf, kb, vb, Ck, Cv = E.setup("mid")          # 2 layers: one layer per shard
    shape = (spec.layers, spec.kv_heads, spec.head_dim)
    hd = spec.kv_heads * spec.head_dim
    groups = E.mid_plan_groups()
    Kc, Vc = E.caches("mid", tokens, pos0)
    m = tokens - 132
    for which, ob, cache in ((0, kb, Kc), (1, vb, Vc)):
        B = K.Basis.create(shape, which, ob.mu, ob.V, ob.sigma, inv_freq=invf if which == 0 else None)
        Pl = K.Plan.create(ob.r, groups)
        unrope = which == 0
        cache_d = cache.cuda()
        # the joint projection on one device, and the shards' partials
        Xfull = K.gather(K.KVView(cache_d, pos0=pos0), 4, m, unrope, invf.astype(np.float32), 0)
        ncols = sum(z for (_, z, _) in groups)
        Dfull = K.project(B, Pl, Xfull, ncols)
        Psum = torch.zeros_like(Dfull)
        cols = np.concatenate([np.arange(s0, s0 + z) for (s0, z, _) in groups])
        Xn_full = _bf16_np(Xfull)
        for g in range(spec.layers):
            sh = JointShard(K, B, Pl, g, g + 1)
            view_g = K.KVView(cache_d[g:g + 1].contiguous(), pos0=pos0)
            Pg = sh.partial(view_g, 4, m, unrope, invf.astype(np.float32), 0, add_bias=(g == 0))
            # each shard's partial vs the oracle's (fp64) partial of the same rows
            ref_g = OPCA.project_partial(ob, Xn_full[:, g * hd:(g + 1) * hd], g * hd, (g + 1) * hd, g == 0, cols)
            assert np.abs(Pg.cpu().numpy() - ref_g).max() <= 2e-5 * np.abs(ref_g).max()
            Psum += Pg
        torch.cuda.synchronize()
        scale = float(Dfull.abs().max())
        assert float((Psum - Dfull).abs().max()) <= 2e-5 * scale          # fp32 sums in another order
        # codes of the summed partials vs the oracle's fp64 projection of the joint features
        payload = K.quantize_pack(Pl, Psum.contiguous())
        pb = payload.cpu().numpy().tobytes()
        Xn = Xn_full
        D_ref = OPCA.project(ob, Xn, cols)
        E.assert_codes_parity(pb, groups, D_ref, m, Xn, ob, cols, f"joint stream={which}")
        # decompression by shard: each shard rebuilds its own layer from the gathered D^
        sh_all = [JointShard(K, B, Pl, g, g + 1) for g in range(spec.layers)]
        section = K.deflate(payload)
        out = torch.zeros_like(cache_d)
        for g, sh in enumerate(sh_all):
            layer_out = [out[g]]
            sh.decompress(section, m, m, 4, layer_out, pos0=pos0)
        torch.cuda.synchronize()
        # oracle: unpack -> dequantise (R5) -> X^ = D^ V_d^T + mu -> RoPE (keys) -> bf16
        shs, scs, cds = OL.unpack(groups, pb, m)
        Dh = np.zeros((m, ob.r))
        for g, (s0, z, t) in enumerate(groups):
            Dh[:, s0:s0 + z] = ON.f16(OQ.dequantize_rows(np.array(shs[g]), np.array(scs[g]), np.array(cds[g]), t))
        Xh = (Dh @ ob.Vd.T + ob.mu[None, :]).reshape(m, spec.layers, spec.kv_heads, spec.head_dim).transpose(1, 0, 2, 3)
        ref = OR.rope_apply_r7(Xh, pos0 + 4 + np.arange(m), invf, 0) if which == 0 else ON.bf16(Xh)
        got = _bf16_np(out[:, 4:4 + m])
        rel = np.linalg.norm(got - ref) / np.linalg.norm(ref)
        assert rel < 1e-3, rel
        assert int((out[:, :4] != 0).sum()) == 0                          # only the middle rows are written


def test_joint_more_accurate_than_per_shard(K):
    """compressing the shards jointly is more accurate than per shard.
    Same target CR (so the same bits per token in total), GPU calibration + DP
    for the joint basis and for each shard's own basis; relative L2 error of the
    decompressed middle tokens."""
    from kvtc_inputs import generate, sample_positions
    spec = E.setup("mid")[0]
    invf = spec.inv_freq().numpy().astype(np.float32)
    tcal = 3200
    samples = sample_positions([tcal], 3000, sinks=4, seed=3)
    t = 1500
    errs = {}
    for which in (0, 1):
        cal = generate(spec, which, tcal, conversation=900, device="cuda")
        x = generate(spec, which, t, conversation=901, device="cuda")
        unrope = which == 0
        rope = invf if unrope else None

        def roundtrip(bcal, bx, lb, le):
            shape = tuple(bx.shape[i] for i in (0, 2, 3))
            basis = K.calibrate([K.KVView(bcal)], samples, which, 10000, inv_freq=rope)
            plan = K.allocate_bits(basis, [K.KVView(bcal)], samples, 16.0)
            X = K.gather(K.KVView(bx), 4, t - 132, unrope, rope, 0)
            ncols = sum(z for (_, z, _) in plan.info().groups)
            payload = K.quantize_pack(plan, K.project(basis, plan, X, ncols).contiguous())
            Dh = K.dequantize(plan, payload, t - 132)
            out = torch.zeros_like(bx)
            K.reconstruct(basis, plan, Dh, t - 132, 4, 0, shape[0], K.KVView(out))
            torch.cuda.synchronize()
            return out[:, 4:t - 128].float()

        joint = roundtrip(cal, x, 0, spec.layers)
        shards = torch.cat([roundtrip(cal[g:g + 1].contiguous(), x[g:g + 1].contiguous(), 0, 1)
                            for g in range(spec.layers)], dim=0)
        ref = x[:, 4:t - 128].float()
        e_joint = float((joint - ref).norm() / ref.norm())
        e_shard = float((shards - ref).norm() / ref.norm())
        errs[which] = (e_joint, e_shard)
        print(f"\n[joint] stream={which} rel L2 joint={e_joint:.4e} per-shard={e_shard:.4e}")
        assert e_joint < e_shard, (e_joint, e_shard)
