"""Diagnostic: independent GPU vs oracle trajectory on the tiny config."""
import os, sys, dataclasses
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]
import oracle_py as O, oracle_model
from paper_2508_21706_b200.engine import TINY, VerifyEngine
B, N, PREFIX = 4, 5, 1024
for lm_scale, router_scale in [(8.0, 4.0), (1.0, 1.0), (32.0, 16.0)]:
    shape = dataclasses.replace(TINY, seed=0x5EED + 1, lm_scale=lm_scale, router_scale=router_scale)
    s_max = PREFIX + N + 64
    eng = VerifyEngine(shape, max_batch=B, max_verify=N, max_seq=s_max, debug=True)
    prefix = np.array([PREFIX, PREFIX - 7, 300, 1], np.int32)
    eng.fill_prefix(prefix)
    om = oracle_model.OracleModel(shape)
    rng = np.random.default_rng(7)
    tokens = rng.integers(0, shape.vocab, size=(B, N)).astype(np.int32)
    res = eng.verify(tokens, prefix)
    x = O.bf16_to_f32(om.embed()[tokens.ravel()]).reshape(B * N, -1).astype(np.float32)
    for l in range(shape.n_layers):
        kc = om.kv_prefix(l, 0, prefix, s_max); vc = om.kv_prefix(l, 1, prefix, s_max)
        x, inter = om.layer(l, x, kc, vc, prefix, N)
        gids = eng.debug_tensor("ids", l, (B * N, 2), np.int32)
        gx = eng.debug_tensor("x_out", l, (B * N, shape.hidden), np.float32)
        glg = eng.debug_tensor("logits_r", l, (B * N, shape.n_expert), np.float32)
        srt = np.sort(inter["logits_r"], axis=1)
        gap = srt[:, -2] - srt[:, -3]
        ga = eng.debug_tensor("attn", l, (B * N, 8, 64), np.uint16)
        print(f"L{l}: id mismatch rows {np.sum(np.any(gids != inter['ids'], axis=1))}, x rel err {np.linalg.norm(gx-x)/np.linalg.norm(x):.2e}, "
              f"attn rel {np.linalg.norm(O.bf16_to_f32(ga)-O.bf16_to_f32(inter['attn']))/np.linalg.norm(O.bf16_to_f32(inter['attn'])):.2e}, "
              f"router logit max err {np.abs(glg-inter['logits_r']).max():.2e}, min gap {gap.min():.2e}, logit std {inter['logits_r'].std():.2f}")
    _, logits = om.head(x)
    gl = eng.debug_tensor("logits", -1, (B * N, shape.vocab), np.float32)
    srt = np.sort(logits, axis=1)
    margin = srt[:, -1] - srt[:, -2]
    row_err = np.abs(gl - logits).max(axis=1)
    print(f"lm={lm_scale} r={router_scale}: logit std {logits.std():.2f}, margins {np.round(margin,3)}, row err {np.round(row_err,3)}")
    print("  argmax equal:", np.mean(np.argmax(gl, 1) == np.argmax(logits, 1)))
    eng.close()
