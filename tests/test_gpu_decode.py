"""GPU: the KV lifecycle and decode loop around the verify step (SURVEY.md §8
f1/f2): layer-major chunked prefill, drafter, draft -> verify -> accept ->
commit on device.

The oracle is greedy autoregressive decoding by the CPU restatement
(tests/oracle_model.OracleDecoder). Under greedy verification every committed
token of ANY speculative decode is the target's greedy token given the
history — acceptance only decides how many tokens a step commits
(specdec.hpp:57-85 with the draw replaced by argmax). The
oracle walks along the GPU's own committed sequence (teacher forcing), so one
near-tie cannot derail the comparison: positions whose oracle top-1/top-2
logit margin is below MARGIN (bf16 noise) only need to be within that margin
(margin screening as in SURVEY.md §7.5).
"""
import dataclasses

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

MARGIN = 0.05  # top-1 minus top-2 logit, in units of the row's logit std
PROMPTS = [70, 33, 5]  # ragged prompt lengths (chunks of C = 32 rows for g = 4)


def _shape():
    from paper_2508_21706_b200.engine import TINY
    return dataclasses.replace(TINY, seed=0x5EED + 7, lm_scale=8.0, router_scale=4.0, draft_layers=1,
                               draft_inter=512)


def _chunk(s):
    return max(1, min(64, 128 // (s.n_q_heads // s.n_kv_heads)))


def _prompts(s):
    rng = np.random.default_rng(11)
    return [rng.integers(0, s.vocab, size=L).astype(np.int32) for L in PROMPTS]


@pytest.fixture(scope="module")
def ref(cuda):
    """Oracle greedy continuations (+ margins) of the test prompts."""
    import oracle_model
    s = _shape()
    om = oracle_model.OracleModel(s)
    s_max = 256
    out = []
    for p in _prompts(s):
        dec = oracle_model.OracleDecoder(om, s_max)
        toks, margins = dec.greedy(p, 0, _chunk(s))
        out.append((toks, margins))
    return s, om, out


def _engine(s, n_max=6, debug=False, attn_cpu=False):
    from paper_2508_21706_b200.engine import VerifyEngine
    return VerifyEngine(s, max_batch=len(PROMPTS), max_verify=n_max, max_seq=256, debug=debug, attn_cpu=attn_cpu)


def test_prefill_matches_oracle(ref, oracle):
    import oracle_model
    s, om, out = ref
    eng = _engine(s, debug=True)
    prompts = _prompts(s)
    nxt = eng.prefill(prompts)
    for r, (toks, margins) in enumerate(out):
        if margins[0] >= MARGIN:
            assert nxt[r] == toks[0], f"request {r}: prefill next token {nxt[r]} != oracle {toks[0]}"
    # K/V written by the chunked prefill vs the oracle's (teacher-forced per chunk)
    f32 = oracle.bf16_to_f32
    d, nkv = s.head_dim, s.n_kv_heads
    for r, p in enumerate(prompts):
        dec = oracle_model.OracleDecoder(om, 256)
        dec.prefill(list(p), _chunk(s))
        for l in range(s.n_layers):
            kc = eng.debug_tensor("k_cache", l, (len(PROMPTS), nkv, 256, d), np.uint16)
            vc = eng.debug_tensor("v_cache", l, (len(PROMPTS), nkv, 256, d), np.uint16)
            for got, exp, nm in ((kc, dec.kc[l], "K"), (vc, dec.vc[l], "V")):
                g = f32(got[r, :, :len(p)]).astype(np.float64)
                e = f32(exp[0, :, :len(p)]).astype(np.float64)
                err = np.sqrt(np.mean((g - e) ** 2) / np.mean(e ** 2))
                assert err < 2e-2, f"request {r} layer {l} {nm}: rel-RMS {err:.3e}"
    # the drafter's K/V over the same prompt (dense layers, oracle restated)
    dw = oracle_model.draft_weights(om, 0)
    for r, p in enumerate(prompts):
        kc = np.zeros((1, nkv, 256, d), np.uint16)
        vc = np.zeros_like(kc)
        C = _chunk(s)
        for c in range(0, len(p), C):
            x = f32(om.embed()[p[c:c + C]]).astype(np.float32)
            oracle_model.attn_block(om, x, dw[0], dw[1], kc, vc, np.array([c], np.int32), len(p[c:c + C]))
        got = eng.debug_tensor("draft_k_cache", 0, (len(PROMPTS), nkv, 256, d), np.uint16)
        g = f32(got[r, :, :len(p)]).astype(np.float64)
        e = f32(kc[0, :, :len(p)]).astype(np.float64)
        err = np.sqrt(np.mean((g - e) ** 2) / np.mean(e ** 2))
        assert err < 1e-2, f"request {r} drafter K: rel-RMS {err:.3e}"
    eng.close()


def _assert_greedy(lg, tok, where):
    """tok must be the argmax of the oracle logits row lg; where the top-1 /
    top-2 margin is below MARGIN (a bf16-noise tie) it must be within it."""
    top = int(np.argmax(lg))
    std = float(np.std(lg))
    if (lg[top] - np.sort(lg)[-2]) / std >= MARGIN:
        assert tok == top, f"{where}: committed {tok} != oracle greedy {top}"
        return 1
    assert lg[tok] >= lg[top] - MARGIN * std, f"{where}: committed {tok} is not a near-tie of {top}"
    return 0


def _teacher_forced(om, prompt, root, committed, where):
    """Walk the oracle along the GPU's own sequence: the prefill's next token
    (root) and every committed token must be the oracle's greedy choice given
    everything before it. Returns the number of decisive checks."""
    import oracle_model
    dec = oracle_model.OracleDecoder(om, 256)
    lg = dec.prefill(list(prompt), _chunk(om.s))
    ok = 0
    for i, tok in enumerate([int(root)] + [int(t) for t in committed]):
        ok += _assert_greedy(lg, tok, f"{where} token {i}")
        lg = dec.run([tok])[-1]
    return ok


@pytest.mark.parametrize("placement", ["gpu", "cpu"])
def test_decode_planted_drafts_commit_greedy_sequence(ref, placement):
    """Planted drafts = the oracle's next k greedy tokens (from the GPU's own
    committed state) corrupted from a random index on: each step must accept
    exactly the uncorrupted prefix, and every committed token is greedy.
    placement "cpu": AttentionPlacement::CPU — target K/V in pinned host DRAM,
    prefill and verify attention on the host pool."""
    import copy
    import oracle_model
    s, om, _ = ref
    b, k = len(PROMPTS), 4
    prompts = _prompts(s)
    eng = _engine(s, attn_cpu=placement == "cpu")
    nxt = eng.prefill(prompts)
    decs, lgs = [], []
    for r, p in enumerate(prompts):  # oracle state after prompt + root
        dec = oracle_model.OracleDecoder(om, 256)
        lg = dec.prefill(list(p), _chunk(s))
        _assert_greedy(lg, int(nxt[r]), f"request {r} prefill")
        decs.append(dec)
        lgs.append(dec.run([int(nxt[r])])[-1])
    rng = np.random.default_rng(5)
    pos = np.zeros(b, np.int64)
    seen = set()
    for step in range(8):
        drafts = np.zeros((b, k), np.int32)
        cut = rng.integers(0, k + 1, size=b)  # first corrupted draft index (k: none)
        decisive = np.zeros(b, bool)
        for r in range(b):
            sim, lg, margins = copy.deepcopy(decs[r]), lgs[r], []
            for j in range(k):
                t = int(np.argmax(lg))
                margins.append(oracle_model.OracleDecoder.margin(lg))
                drafts[r, j] = t if j < cut[r] else (t + 1 + j) % s.vocab
                lg = sim.run([t])[-1]
            decisive[r] = all(m >= MARGIN for m in margins[:cut[r]])
        eng.decode_step(k, drafts)
        com, n, kv, root = eng.decode_read(b, 64)
        for r in range(b):
            new = [int(t) for t in com[r, pos[r]:n[r]]]
            if decisive[r]:
                assert len(new) - 1 == cut[r], f"step {step} request {r}: accepted {len(new) - 1} != planted {cut[r]}"
                seen.add(int(cut[r]))
            for i, t in enumerate(new):  # teacher-forced: every committed token is greedy
                _assert_greedy(lgs[r], t, f"step {step} request {r} token {i}")
                lgs[r] = decs[r].run([t])[-1]
            pos[r] = n[r]
        assert np.array_equal(kv, np.array(PROMPTS) + n), "kv_len must advance by the committed count"
        assert np.array_equal(root, com[np.arange(b), n - 1]), "the bonus token becomes the next root"
    assert len(seen) >= 3, f"planted cuts should exercise several acceptance lengths: {seen}"
    eng.close()


@pytest.mark.parametrize("k", [0, 3])
def test_decode_with_drafter_commits_greedy_sequence(ref, k):
    """The on-device drafter proposes (random-init: mostly rejected); k = 0 is
    plain autoregressive decoding. Either way every committed token is the
    target's greedy token given the GPU's own history."""
    s, om, _ = ref
    b, steps = len(PROMPTS), 12
    prompts = _prompts(s)
    eng = _engine(s)
    nxt = eng.prefill(prompts)
    for _ in range(steps):
        eng.decode_step(k)
    com, n, kv, root = eng.decode_read(b, 128)
    assert np.all(n >= steps)
    decisive = sum(_teacher_forced(om, prompts[r], nxt[r], com[r, :n[r]], f"request {r}") for r in range(b))
    assert decisive >= b * steps // 2, f"too few decisive positions ({decisive})"
    t = eng.last_times()
    if k > 0:
        assert t["draft"] > 0.0
    eng.close()


def test_decode_errors(ref):
    s, _, _ = ref
    eng = _engine(s)
    with pytest.raises(ValueError, match="prefill or smo_engine_decode_begin"):
        eng.decode_step(1)
    eng.decode_begin(np.zeros(3, np.int32), np.array([10, 10, 10], np.int32))
    with pytest.raises(ValueError, match="max_verify"):
        eng.decode_step(6)
    eng.close()
    from paper_2508_21706_b200.engine import VerifyEngine
    e2 = VerifyEngine(dataclasses.replace(s, draft_layers=0, draft_inter=0), max_batch=2, max_verify=4, max_seq=64)
    e2.decode_begin(np.zeros(2, np.int32), np.array([3, 4], np.int32))
    with pytest.raises(ValueError, match="drafter"):
        e2.decode_step(2)
    e2.decode_step(2, np.ones((2, 2), np.int32))  # planted drafts need no drafter
    e2.close()


def test_paged_kv_engine_matches_contiguous(ref):
    """Paged K/V: the engine on a page pool (block table
    shared by all layers, pages assigned as requests grow) commits exactly
    what the contiguous layout commits — prefill, drafter and planted-draft
    decoding."""
    from paper_2508_21706_b200.engine import VerifyEngine
    s, _, _ = ref
    b, k = len(PROMPTS), 4
    prompts = _prompts(s)
    rng = np.random.default_rng(9)
    plants = [rng.integers(0, s.vocab, size=(b, k)).astype(np.int32) for _ in range(3)]
    outs = []
    for pages in (0, 6):  # 6 pages of 128 tokens: less than b * ceil(256 / 128)
        eng = VerifyEngine(s, max_batch=b, max_verify=6, max_seq=256, kv_pages=pages)
        nxt = eng.prefill(prompts)
        for d in plants:
            eng.decode_step(k, d)
        for _ in range(3):
            eng.decode_step(3)
        outs.append((nxt, eng.decode_read(b, 64)))
        eng.close()
    (n0, r0), (n1, r1) = outs
    assert np.array_equal(n0, n1)
    for a, c in zip(r0, r1):
        assert np.array_equal(a, c)


def test_paged_kv_pool_exhaustion(ref):
    from paper_2508_21706_b200 import _lib
    from paper_2508_21706_b200.engine import VerifyEngine
    s, _, _ = ref
    eng = VerifyEngine(s, max_batch=3, max_verify=6, max_seq=256, kv_pages=2)
    with pytest.raises(_lib.CapacityError, match="page pool exhausted"):
        eng.prefill(_prompts(s))
    eng.close()


def test_decode_run_cuda_graph(ref):
    """decode_run(graph=True): one captured CUDA graph per iteration (drafter,
    expert streaming on the copy stream, verify, commit) replayed; every
    committed token is still the target's greedy token, and the graph path
    issues one launch per iteration."""
    import torch
    from paper_2508_21706_b200 import _lib
    s, om, _ = ref
    b, k, steps = len(PROMPTS), 3, 6
    prompts = _prompts(s)
    eng = _engine(s)
    nxt = eng.prefill(prompts)
    stream = torch.cuda.Stream()
    eng.decode_run(k, 2, graph=True, stream=stream.cuda_stream)       # captures
    eng.decode_run(k, steps - 2, graph=True, stream=stream.cuda_stream)  # replays the same graph
    stream.synchronize()
    com, n, kv, root = eng.decode_read(b, 128)
    assert np.all(n >= steps)
    assert np.array_equal(kv, np.array(PROMPTS) + n)
    decisive = sum(_teacher_forced(om, prompts[r], nxt[r], com[r, :n[r]], f"graph request {r}") for r in range(b))
    assert decisive >= b * steps // 2
    with pytest.raises(ValueError, match="non-default stream"):
        eng.decode_run(k, 1, graph=True)
    eng.close()


def test_decode_planted_tree_compacts_kv(ref):
    """Tree K/V lifecycle: each step plants a 7-node tree —
    a spine of the oracle's greedy tokens (correct up to a random cut) with a
    decoy sibling at every level, sibling order random. Greedy accept must take
    exactly the spine prefix, and because the next steps attend over the
    COMPACTED K/V (spine rows moved to kv_len + j in every target and drafter
    layer), every later committed token is still the greedy one."""
    import copy
    import oracle_model
    s, om, _ = ref
    b, n = len(PROMPTS), 7
    prompts = _prompts(s)
    eng = _engine(s, n_max=8)
    nxt = eng.prefill(prompts)
    decs, lgs = [], []
    for r, p in enumerate(prompts):
        dec = oracle_model.OracleDecoder(om, 256)
        dec.prefill(list(p), _chunk(s))
        decs.append(dec)
        lgs.append(dec.run([int(nxt[r])])[-1])
    rng = np.random.default_rng(21)
    pos = np.zeros(b, np.int64)
    seen = set()
    for step in range(6):
        tokens = np.zeros((b, n - 1), np.int32)
        parents = np.full((b, n), -1, np.int32)
        cut = rng.integers(0, 4, size=b)
        decisive = np.zeros(b, bool)
        for r in range(b):
            sim, lg, margins = copy.deepcopy(decs[r]), lgs[r], []
            spine_parent, node = 0, 1
            for lvl in range(3):
                g = int(np.argmax(lg))
                margins.append(oracle_model.OracleDecoder.margin(lg))
                spine_tok = g if lvl < cut[r] else (g + 7 + lvl) % s.vocab
                decoy_tok = (g + 1 + lvl) % s.vocab
                order = [("spine", spine_tok), ("decoy", decoy_tok)]
                if rng.integers(0, 2):
                    order.reverse()
                spine_node = None
                for kind, tok in order:
                    tokens[r, node - 1] = tok
                    parents[r, node] = spine_parent
                    if kind == "spine":
                        spine_node = node
                    node += 1
                spine_parent = spine_node
                lg = sim.run([g])[-1]
            decisive[r] = all(m >= MARGIN for m in margins[:cut[r]])
        eng.decode_step_tree(tokens, parents)
        com, cnt, kv, root = eng.decode_read(b, 64)
        for r in range(b):
            new = [int(t) for t in com[r, pos[r]:cnt[r]]]
            if decisive[r]:
                assert len(new) - 1 == cut[r], f"step {step} request {r}: accepted {len(new) - 1} != {cut[r]}"
                seen.add(int(cut[r]))
            for i, t in enumerate(new):
                _assert_greedy(lgs[r], t, f"tree step {step} request {r} token {i}")
                lgs[r] = decs[r].run([t])[-1]
            pos[r] = cnt[r]
        assert np.array_equal(kv, np.array(PROMPTS) + cnt)
    assert len(seen) >= 2, seen
    # a chain step after the trees still commits greedy tokens (drafter K/V compacted too)
    eng.decode_step(3)
    com, cnt, kv, root = eng.decode_read(b, 64)
    for r in range(b):
        for i, t in enumerate(com[r, pos[r]:cnt[r]]):
            _assert_greedy(lgs[r], int(t), f"post-tree request {r} token {i}")
            lgs[r] = decs[r].run([int(t)])[-1]
    eng.close()


def test_engine_option_conflicts(ref):
    """Unsupported option mixes fail loudly at creation, with the reason."""
    from paper_2508_21706_b200.engine import VerifyEngine
    s, _, _ = ref
    with pytest.raises(ValueError, match="contiguous host K/V"):
        VerifyEngine(s, max_batch=2, max_verify=4, max_seq=256, attn_cpu=True, kv_pages=-1)


def test_paged_graph_decode_matches_paged_eager(ref):
    """decode_run(graph=True) maps every page the run needs before replaying;
    on a paged pool it commits what the eager paged loop commits."""
    import torch
    from paper_2508_21706_b200.engine import VerifyEngine
    s, _, _ = ref
    b, k, steps = len(PROMPTS), 3, 5
    out = []
    stream = torch.cuda.Stream()
    for graph in (False, True):
        eng = VerifyEngine(s, max_batch=b, max_verify=6, max_seq=256, kv_pages=-1)
        eng.prefill(_prompts(s), stream=stream.cuda_stream)
        eng.decode_run(k, steps, graph=graph, stream=stream.cuda_stream)
        stream.synchronize()
        out.append(eng.decode_read(b, 64))
        eng.close()
    for a, c in zip(out[0], out[1]):
        assert np.array_equal(a, c)


@pytest.mark.parametrize("g", [1, 0])
def test_drafter_cpu_split_commits_greedy_sequence(ref, g):
    """Drafter CPU part: requests [g, b) keep their drafter
    K/V in pinned host memory and attend on the host pool while K1 attends
    the GPU part. Greedy verification makes the committed tokens independent
    of where the drafter attended: identical to an all-GPU engine; the split
    measures a host attention time per drafter step."""
    from paper_2508_21706_b200.engine import VerifyEngine as _VE
    s, om, _ = ref
    b, steps, k = len(PROMPTS), 8, 3
    prompts = _prompts(s)
    out = {}
    for split in (False, True):
        eng = _VE(s, max_batch=b, max_verify=6, max_seq=256, draft_cpu_kv=split)
        nxt = eng.prefill(prompts)
        if split:
            eng.set_draft_split(g)
        times = []
        for _ in range(steps):
            eng.decode_step(k)
            if split:
                times.append(eng.draft_split_times())
        out[split] = (nxt, eng.decode_read(b, 128))
        eng.close()
        if split:
            for t in times:
                assert t.shape == (k + 1, 3) and np.all(t[:, 1] > 0) and np.all(t >= 0)
    (n0, (c0, m0, kv0, _)), (n1, (c1, m1, kv1, _)) = out[False], out[True]
    assert np.array_equal(n0, n1)
    for r in range(b):
        m = min(m0[r], m1[r])
        assert m >= steps and np.array_equal(c0[r, :m], c1[r, :m]), r
