"""Prefill + decode on a mid-size shape (d=128, Mixtral head layout) — a
quick GPU check outside pytest; run under compute-sanitizer to localise
faults. usage: python tools/dbg_prefill.py [mid|mixtral] [b] [L]"""
import dataclasses
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_21706_b200.engine import MIXTRAL_8X7B, ModelShape, VerifyEngine  # noqa: E402

kind = sys.argv[1] if len(sys.argv) > 1 else "mid"
b = int(sys.argv[2]) if len(sys.argv) > 2 else 4
L = int(sys.argv[3]) if len(sys.argv) > 3 else 100
if kind == "mid":
    s = ModelShape(hidden=1024, inter=2048, n_expert=8, top_k=2, n_layers=2, n_q_heads=32, n_kv_heads=8,
                   head_dim=128, vocab=32000, draft_layers=1, draft_inter=1024)
else:
    s = dataclasses.replace(MIXTRAL_8X7B, draft_layers=1, draft_inter=14336)
eng = VerifyEngine(s, max_batch=b, max_verify=9, max_seq=L + 128, host_alias_layers=2 if kind != "mid" else 0)
rng = np.random.default_rng(0)
nxt = eng.prefill(rng.integers(0, s.vocab, size=(b, L)).astype(np.int32))
print("prefill ok", nxt[:4], eng.last_times(), flush=True)
for k in (0, 4, 8):
    eng.decode_step(k)
com, n, kv, root = eng.decode_read(b, 32)
print("decode ok", n, kv, eng.last_times(), flush=True)
