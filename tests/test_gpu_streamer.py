"""The standalone expert streamer (smo_streamer_*, csrc/streamer.cu): blocks
in pinned host memory reach their HBM slot bit-exactly — raw, unary-coded and
3-bit-coded blocks mixed, hot-cached blocks served from the cache, BATCH_ONE
`active` masks honoured, slots reused only after release (the reference's
H2D_EXPERTS(l) -> GPU_MOE(l) dependency, pipeline.hpp:147-206)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _read(ptr, nbytes, stream):
    import torch
    from cuda.bindings import runtime as rt
    out = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    err, = rt.cudaMemcpyAsync(out.data_ptr(), ptr, nbytes, rt.cudaMemcpyKind.cudaMemcpyDeviceToDevice, stream)
    assert err == rt.cudaError_t.cudaSuccess
    return out


def test_streamer_layers_bit_exact(cuda):
    import torch
    from paper_2508_21706_b200 import ops
    L, E, vals = 5, 3, 64 * 1024
    blk = 2 * vals
    g = torch.Generator(device="cuda").manual_seed(3)
    raw, host, codes = [], [], []
    for i in range(L * E):
        x = ((torch.rand(vals, generator=g, device="cuda") * 2 - 1) * 0.02).to(torch.bfloat16)
        raw.append(x.view(torch.uint8).clone())
        code = [0, 1, 3][i % 3]
        if code:
            c, ovf = ops.expert_encode(x, code)
            assert not ovf
            src = c.cpu()
        else:
            src = x.view(torch.uint8).cpu()
        h = torch.empty(src.numel(), dtype=torch.uint8).pin_memory()
        h.copy_(src)
        host.append(h)
        codes.append(code)
    s = ops.ExpertStreamer(host, L, E, blk, codes=codes, hbm_slots=2, cache_bytes=2 * blk)
    st = torch.cuda.Stream()
    try:
        for rep in range(2):  # the slots cycle through the layers twice
            for layer in range(L):
                active = None if layer != 3 else [True, False, True]  # BATCH_ONE-style mask
                s.enqueue_layer(layer, active)
                s.wait_layer(layer, st.cuda_stream)
                got = [_read(s.expert_ptr(layer, e), blk, st.cuda_stream) for e in range(E)]
                s.release_layer(layer, st.cuda_stream)
                st.synchronize()
                for e in range(E):
                    i = layer * E + e
                    if active is not None and not active[e] and i >= 2:
                        continue  # not streamed (and not cached): slot content unspecified
                    assert torch.equal(got[e], raw[i]), (rep, layer, e, codes[i])
        assert s.ready_event(L - 1) != 0
    finally:
        s.close()


def test_streamer_rejects_bad_args(cuda):
    import torch
    from paper_2508_21706_b200 import _lib as Lb
    from paper_2508_21706_b200 import ops
    h = torch.empty(4096, dtype=torch.uint8).pin_memory()
    with pytest.raises((ValueError, Lb.SmoError)):
        ops.ExpertStreamer([h], 1, 1, 4096, hbm_slots=1)  # needs >= 2 slots
    with pytest.raises((ValueError, Lb.SmoError)):
        ops.ExpertStreamer([h], 1, 1, 4096, codes=[2])  # unknown code
