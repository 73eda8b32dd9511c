"""GPU tier: the T2 tile code (tcode.cu) and the fused coded expert kernel.

* the GPU encoder writes exactly the bytes of the numpy restatement
  (tests/tcode_ref.py) and both decoders invert it, on uniform-init,
  gaussian-like and arbitrary bit patterns;
* a whole Mixtral expert block (176 M values) round-trips bit for bit;
* K4-MoE on coded experts (smo_moe_experts_coded, decode in shared memory)
  is BIT-IDENTICAL to K4-MoE on the decoded bf16 weights (same tiles, same
  MMA order), at a small shape with ragged groups and at the bench's launch
  (576 rows x 8 Mixtral experts)."""
import math

import numpy as np
import pytest

import tcode_ref as T

pytestmark = pytest.mark.gpu


def _block(torch, cuda, kind, h, hi, seed=0x5EED, base=1100):
    from paper_2508_21706_b200 import ops
    blk = torch.empty(3 * h * hi, dtype=torch.bfloat16, device=cuda)
    if kind == "wide":
        g = torch.Generator(device="cpu").manual_seed(seed)
        bits = torch.randint(0, 1 << 16, (3 * h * hi,), generator=g, dtype=torch.int32)
        bits[::7] = 0
        bits[5::11] = 0x0001  # denormals (exponent 0 with a mantissa)
        return bits.to(torch.int16).view(torch.bfloat16).to(cuda)
    fill = ops.fill_uniform_ if kind == "uniform" else ops.fill_normal_
    fill(blk[:hi * h], seed, base, math.sqrt(3.0 / h))
    fill(blk[hi * h:2 * hi * h], seed, base + 1, math.sqrt(3.0 / h))
    fill(blk[2 * hi * h:], seed, base + 2, math.sqrt(3.0 / hi))
    return blk


def _u16(torch, t):
    return t.view(torch.int16).cpu().numpy().view(np.uint16)


@pytest.mark.parametrize("kind", ["uniform", "gaussian", "wide"])
def test_tcode_gpu_encoder_matches_numpy(cuda, kind):
    import torch
    from paper_2508_21706_b200 import ops
    h, hi = 256, 384
    blk = _block(torch, cuda, kind, h, hi)
    code = ops.tcode_encode(blk, h, hi)
    ref = T.encode_expert(_u16(torch, blk), h, hi)
    assert code.numel() == len(ref)
    assert bytes(code.cpu().numpy().tobytes()) == ref
    out = ops.tcode_decode(code, h, hi)
    assert torch.equal(out.view(torch.int16), blk.view(torch.int16))


def test_tcode_full_mixtral_block(cuda):
    """One whole Mixtral expert block through the tile code: bit-exact round
    trip; ~10.4 bits/weight; sampled tiles decode identically in numpy."""
    import torch
    from paper_2508_21706_b200 import ops
    h, hi = 4096, 14336
    blk = _block(torch, cuda, "uniform", h, hi, base=1100)
    code = ops.tcode_encode(blk, h, hi)
    bpw = code.numel() * 8 / blk.numel()
    assert 10.2 < bpw < 10.6, bpw
    out = ops.tcode_decode(code, h, hi)
    assert torch.equal(out.view(torch.int16), blk.view(torch.int16))
    del out
    c = code.cpu().numpy()
    nt = 3 * h * hi // (128 * 64)
    toff = c[:4 * (nt + 1)].view("<u4")
    xs = _u16(torch, blk)
    for t in (0, 1, nt // 3, nt // 2 + 5, nt - 1):
        m, tl = divmod(t, nt // 3)
        R, C = (hi, h) if m < 2 else (h, hi)
        nb, kb = divmod(tl, C // 64)
        W = xs[m * h * hi:(m + 1) * h * hi].reshape(R, C)
        tile = T.decode_tile(c[toff[t]:toff[t + 1]])
        assert np.array_equal(tile, W[nb * 128:(nb + 1) * 128, kb * 64:(kb + 1) * 64]), t


def _coded_vs_plain(torch, cuda, h, hi, E, rows_per, kind, splits=0, fmt=2):
    from paper_2508_21706_b200 import ops
    g = torch.Generator(device=cuda).manual_seed(7)
    blks = [_block(torch, cuda, kind, h, hi, base=2000 + 3 * e) for e in range(E)]
    pool = torch.cat(blks)
    codes = [ops.tcode_encode(b, h, hi, fmt=fmt) for b in blks]
    w_code = torch.tensor([c.data_ptr() for c in codes], dtype=torch.int64, device=cuda)
    counts = torch.tensor(rows_per, dtype=torch.int32)
    off = torch.zeros(E + 1, dtype=torch.int32)
    off[1:] = torch.cumsum(counts, 0)
    rows = int(off[-1])
    off = off.to(cuda)
    x = (torch.rand((rows, h), generator=g, device=cuda) * 2 - 1).to(torch.bfloat16)
    blk = 3 * h * hi
    h0, y0 = ops.moe_experts(x, off, pool, h=h, h_i=hi, n_expert=E, w_block_stride=blk * 2, w_pool_blocks=E,
                             splits=splits)
    h1, y1 = ops.moe_experts_coded(x, off, w_code, h=h, h_i=hi, n_expert=E, splits=splits, fmt=fmt)
    torch.cuda.synchronize()
    assert y0.shape == y1.shape
    assert torch.equal(h0.view(torch.int16), h1.view(torch.int16))
    assert torch.equal(y0.view(torch.int32), y1.view(torch.int32))
    if kind == "wide":  # NaN / Inf bit patterns: bit identity is the whole check
        return
    # and the plain kernel itself against fp32 torch on the first non-empty expert
    e = int(np.flatnonzero(np.asarray(rows_per) > 0)[0])
    a, b = int(off[e]), int(off[e + 1])
    w1 = pool[e * blk:e * blk + hi * h].view(hi, h).float()
    w3 = pool[e * blk + hi * h:e * blk + 2 * hi * h].view(hi, h).float()
    gg, uu = x[a:b].float() @ w1.T, x[a:b].float() @ w3.T
    H = gg * torch.sigmoid(gg) * uu
    assert (h1[a:b].float() - H).abs().max().item() <= 2 ** -7 * max(1.0, H.abs().max().item())


@pytest.mark.parametrize("kind", ["uniform", "gaussian", "wide"])
def test_moe_coded_bit_identical_small(cuda, kind):
    import torch
    # ragged groups incl. an empty expert and one above 128 rows
    _coded_vs_plain(torch, cuda, 512, 768, 6, [5, 0, 33, 130, 1, 64], kind)


def test_moe_coded_bit_identical_splits(cuda):
    import torch
    for sp in (1, 2, 4):
        _coded_vs_plain(torch, cuda, 256, 512, 3, [17, 40, 9], "uniform", splits=sp)


def test_moe_coded_bit_identical_mixtral_dims(cuda):
    """The bench's launch: 576 (token, slot) rows over 8 experts at h 4096,
    h_i 14336 (even-ish routing), production split."""
    import torch
    rows = [70, 75, 68, 80, 71, 69, 72, 71]
    _coded_vs_plain(torch, cuda, 4096, 14336, 8, rows, "uniform")


# ---------------------------------------------------------------- T3
import tcode3_ref as T3  # noqa: E402


@pytest.mark.parametrize("kind", ["uniform", "gaussian", "wide"])
def test_tcode3_gpu_encoder_matches_numpy(cuda, kind):
    """T3: the GPU encoder writes exactly the numpy restatement's bytes
    (tests/tcode3_ref.py) and the GPU decoder inverts it bit for bit."""
    import torch
    from paper_2508_21706_b200 import ops
    h, hi = 256, 384
    blk = _block(torch, cuda, kind, h, hi)
    code = ops.tcode_encode(blk, h, hi, fmt=3)
    ref = T3.encode_expert(_u16(torch, blk), h, hi)
    assert code.numel() == len(ref)
    assert bytes(code.cpu().numpy().tobytes()) == ref
    out = ops.tcode_decode(code, h, hi, fmt=3)
    assert torch.equal(out.view(torch.int16), blk.view(torch.int16))


def test_tcode3_full_mixtral_block(cuda):
    """A whole Mixtral expert block through T3: bit-exact, ~11.2 bits/weight."""
    import torch
    from paper_2508_21706_b200 import ops
    h, hi = 4096, 14336
    blk = _block(torch, cuda, "uniform", h, hi, base=1100)
    code = ops.tcode_encode(blk, h, hi, fmt=3)
    bpw = code.numel() * 8 / blk.numel()
    assert 11.0 < bpw < 11.4, bpw
    out = ops.tcode_decode(code, h, hi, fmt=3)
    assert torch.equal(out.view(torch.int16), blk.view(torch.int16))


@pytest.mark.parametrize("kind", ["uniform", "gaussian", "wide"])
def test_moe_coded3_bit_identical_small(cuda, kind):
    import torch
    _coded_vs_plain(torch, cuda, 512, 768, 6, [5, 0, 33, 130, 1, 64], kind, fmt=3)


def test_moe_coded3_bit_identical_mixtral_dims(cuda):
    import torch
    rows = [70, 75, 68, 80, 71, 69, 72, 71]
    _coded_vs_plain(torch, cuda, 4096, 14336, 8, rows, "uniform", fmt=3)


@pytest.mark.parametrize("fmt", [2, 3])
def test_moe_coded_repeat_bit_identical(cuda, fmt):
    """Race detector for the coded expert kernel's decoder-warp / token-ring /
    MMA hand-offs (compute-sanitizer is closed on the GPU pool): repeated
    launches, foreign kernels in between, bit-identical H and y."""
    import torch
    from paper_2508_21706_b200 import ops
    h, hi, E = 512, 768, 6
    rows_per = [5, 0, 33, 130, 1, 64]
    g = torch.Generator(device=cuda).manual_seed(11)
    blks = [_block(torch, cuda, "uniform", h, hi, base=3000 + 3 * e) for e in range(E)]
    codes = [ops.tcode_encode(b, h, hi, fmt=fmt) for b in blks]
    w_code = torch.tensor([c.data_ptr() for c in codes], dtype=torch.int64, device=cuda)
    off = torch.zeros(E + 1, dtype=torch.int32)
    off[1:] = torch.cumsum(torch.tensor(rows_per, dtype=torch.int32), 0)
    rows = int(off[-1])
    off = off.to(cuda)
    x = (torch.rand((rows, h), generator=g, device=cuda) * 2 - 1).to(torch.bfloat16)
    h0, y0 = ops.moe_experts_coded(x, off, w_code, h=h, h_i=hi, n_expert=E, splits=2, fmt=fmt)
    junk = torch.empty(1 << 22, device=cuda)
    outs = []
    for i in range(40):
        if i % 2 == 0:
            junk.normal_()
        outs.append(ops.moe_experts_coded(x, off, w_code, h=h, h_i=hi, n_expert=E, splits=2, fmt=fmt))
    torch.cuda.synchronize()
    for i, (hh, yy) in enumerate(outs):
        assert torch.equal(hh.view(torch.int16), h0.view(torch.int16)), f"launch {i}: H differs"
        assert torch.equal(yy.view(torch.int32), y0.view(torch.int32)), f"launch {i}: y differs"
