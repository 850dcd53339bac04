"""Pins for oracle/model.py against library routines and closed forms."""
import numpy as np
import torch
import torch.nn.functional as F

from oracle import model
from oracle.numerics import round_bf16


def _rng(s=0):
    return np.random.default_rng(s)


def test_attention_matches_torch_sdpa_gqa_causal_chain():
    """Chain row j sees all L cache keys + chain keys 0..j; GQA head hq -> hq // G."""
    rng = _rng(1)
    L, R, Hq, Hkv, dh = 37, 5, 8, 2, 16
    q = rng.standard_normal((R, Hq, dh))
    ck, cv = rng.standard_normal((L, Hkv, dh)), rng.standard_normal((L, Hkv, dh))
    kk, vv = rng.standard_normal((R, Hkv, dh)), rng.standard_normal((R, Hkv, dh))
    got = model.verify_attention(q, ck, cv, kk, vv)
    # torch: dense keys, boolean mask, kv heads expanded with repeat_interleave
    K = torch.tensor(np.concatenate([ck, kk])).permute(1, 0, 2)          # [Hkv, L+R, dh]
    Vt = torch.tensor(np.concatenate([cv, vv])).permute(1, 0, 2)
    K = K.repeat_interleave(Hq // Hkv, dim=0)
    Vt = Vt.repeat_interleave(Hq // Hkv, dim=0)
    Q = torch.tensor(q).permute(1, 0, 2)                                 # [Hq, R, dh]
    mask = torch.ones(R, L + R, dtype=torch.bool)
    mask[:, L:] = torch.tril(torch.ones(R, R, dtype=torch.bool))
    ref = F.scaled_dot_product_attention(Q, K, Vt, attn_mask=mask)       # [Hq, R, dh]
    ref = ref.permute(1, 0, 2).reshape(R, Hq * dh).numpy()
    assert np.array_equal(got, round_bf16(ref)) or np.max(np.abs(got - round_bf16(ref))) <= \
        2.0 ** -7 * np.max(np.abs(ref))
    # almost all elements identical after rounding (differences only at exact rounding ties)
    assert np.mean(got == round_bf16(ref)) > 0.999


def test_attention_single_key_returns_value():
    rng = _rng(2)
    q = rng.standard_normal((1, 4, 8))
    v = round_bf16(rng.standard_normal((1, 2, 8)))
    out = model.verify_attention(q, np.zeros((0, 2, 8)), np.zeros((0, 2, 8)),
                                 rng.standard_normal((1, 2, 8)), v)
    assert np.array_equal(out.reshape(4, 8), np.repeat(v[0], 2, axis=0))


def test_softmax_matches_torch():
    x = _rng(3).standard_normal((7, 300)) * 10
    ref = torch.log_softmax(torch.tensor(x), dim=-1).exp().numpy()
    assert np.allclose(model.softmax(x), ref, rtol=1e-13, atol=0)


def test_rmsnorm_closed_form_and_torch():
    D, eps = 64, 1e-5
    for c in (0.3, -2.0, 1e-3):
        x = np.full((1, D), c)
        assert np.allclose(model.rmsnorm(x, 1.0, eps), c / np.sqrt(c * c + eps), rtol=1e-15)
    x = _rng(4).standard_normal((5, D))
    g = _rng(5).standard_normal(D)
    ref = F.rms_norm(torch.tensor(x), (D,), weight=torch.tensor(g), eps=eps).numpy()
    assert np.allclose(model.rmsnorm(x, g, eps), ref, rtol=1e-13, atol=1e-15)


def test_rope_table_definition():
    cos, sin = model.rope_table(64, 16, 10000.0)
    assert cos.dtype == np.float32 and cos.shape == (64, 8)
    assert np.all(cos[0] == 1) and np.all(sin[0] == 0)
    # m = 0 rotates by exactly pos radians; m = 1 by pos * theta^(-2/16)
    assert cos[5, 0] == np.float32(np.cos(5.0))
    assert sin[7, 1] == np.float32(np.sin(7.0 * 10000.0 ** (-2.0 / 16)))


def test_rope_matches_complex_rotation():
    """rotate_half pairs (m, m + d/2) as a complex number rotated by e^{i pos w_m}."""
    rng = _rng(6)
    dh, R, H = 32, 6, 3
    cos, sin = model.rope_table(100, dh, 500000.0)
    x = rng.standard_normal((R, H, dh))
    pos = np.array([0, 1, 5, 17, 63, 99])
    got = model.rope(x, pos, cos, sin)
    xc = torch.complex(torch.tensor(x[..., : dh // 2]), torch.tensor(x[..., dh // 2:]))
    rot = torch.complex(torch.tensor(cos[pos].astype(np.float64)),
                        torch.tensor(sin[pos].astype(np.float64)))[:, None, :]
    yc = xc * rot
    ref = np.concatenate([yc.real.numpy(), yc.imag.numpy()], axis=-1)
    assert np.allclose(got, ref, rtol=0, atol=1e-13)
    # pair norms preserved up to the fp32 table's |cos^2 + sin^2 - 1|
    n0 = x[..., : dh // 2] ** 2 + x[..., dh // 2:] ** 2
    n1 = got[..., : dh // 2] ** 2 + got[..., dh // 2:] ** 2
    assert np.allclose(n0, n1, rtol=1e-6)


def test_rope_relative_position_property():
    rng = _rng(7)
    dh = 64
    cos, sin = model.rope_table(400, dh, 500000.0)
    q = rng.standard_normal((1, 1, dh))
    k = rng.standard_normal((1, 1, dh))
    d1 = np.sum(model.rope(q, np.array([50]), cos, sin) * model.rope(k, np.array([20]), cos, sin))
    d2 = np.sum(model.rope(q, np.array([330]), cos, sin) * model.rope(k, np.array([300]), cos, sin))
    assert abs(d1 - d2) < 1e-4 * (1 + abs(d1))


def test_silu_and_swiglu_match_torch():
    rng = _rng(8)
    x = rng.standard_normal(1000) * 5
    assert np.allclose(model.silu(x), F.silu(torch.tensor(x)).numpy(), rtol=1e-14, atol=1e-300)
    D, Fd = 16, 12
    b = round_bf16(rng.standard_normal((3, D)))
    W = round_bf16(rng.standard_normal((2 * Fd, D)) * 0.1)
    got = model.swiglu(b, W)
    tb, tW = torch.tensor(b), torch.tensor(W)
    ref = F.silu(tb @ tW[:Fd].T) * (tb @ tW[Fd:].T)
    assert np.array_equal(got, round_bf16(ref.numpy())) or np.mean(got == round_bf16(ref.numpy())) > 0.99


def test_qkv_head_slicing():
    """q head h is rows h*dh..(h+1)*dh of wqkv; k heads follow q heads; v heads follow k heads."""
    rng = _rng(9)
    Hq, Hkv, dh, D = 4, 2, 8, 16
    a = round_bf16(rng.standard_normal((3, D)))
    W = round_bf16(rng.standard_normal(((Hq + 2 * Hkv) * dh, D)))
    cos, sin = model.rope_table(10, dh, 500000.0)
    pos = np.array([0, 0, 0])
    q, k, v = model.qkv_rope(a, W, pos, cos, sin, Hq, Hkv, dh)
    assert np.array_equal(q[:, 3], round_bf16(a @ W[3 * dh:4 * dh].T))
    assert np.array_equal(k[:, 1], round_bf16(a @ W[(Hq + 1) * dh:(Hq + 2) * dh].T))
    assert np.array_equal(v[:, 0], round_bf16(a @ W[(Hq + 2) * dh:(Hq + 3) * dh].T))


def test_tile_stats_vs_torch():
    rng = _rng(10)
    x = rng.standard_normal((3, 1000)) * 4
    x[1, 300] = x[1, 700] = 100.0         # tie across tiles -> lowest index
    x[2, 260] = x[2, 270] = 90.0          # tie inside a tile
    mx, se, am = model.tile_stats(x, tile=256)
    t = torch.tensor(x)
    for tt in range(mx.shape[1]):
        blk = t[:, tt * 256:(tt + 1) * 256]
        assert np.allclose(mx[:, tt], blk.max(dim=1).values.numpy())
        assert np.allclose(np.log(se[:, tt]) + mx[:, tt], torch.logsumexp(blk, dim=1).numpy(), rtol=1e-13)
    assert am[1, 1] == 300 and am[1, 2] == 700 and am[2, 1] == 260


def test_lm_head_chunking_is_plain_product():
    rng = _rng(11)
    z = round_bf16(rng.standard_normal((2, 32)))
    W = round_bf16(rng.standard_normal((100, 32)))
    assert np.allclose(model.lm_head(z, W, chunk=7), (torch.tensor(z) @ torch.tensor(W).T).numpy(),
                       rtol=1e-14, atol=1e-12)
