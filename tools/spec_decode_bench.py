"""Measured speculative-decoding gain on the offloaded Mixtral-8x7B verify
engine (BASELINE config 2 shape, b=32, prompts of 1024 tokens, coded expert
transfer): committed tokens/s of plain greedy decoding (k=0) vs greedy
verification of k=8 drafts whose acceptance follows the reference's chain
model with p=0.8 (specdec.hpp:57-85, workload_apps.json acceptance).

Drafts are PLANTED: the greedy continuation is first produced by k=0
decoding, the state is rebuilt by a second prefill, and every draft position
keeps the true token with probability p (the rest of the chain is corrupted
from the first rejection on), so the accepted lengths are the reference
model's while every committed token is compared with the greedy sequence
(agreement reported: random-init logits have near-ties that bf16
accumulation order can flip). Prints one JSON line."""
import dataclasses
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_21706_b200.engine import MIXTRAL_8X7B, VerifyEngine  # noqa: E402

b, prompt, k, iters, p = 32, 1024, 8, 2, 0.8
shape = dataclasses.replace(MIXTRAL_8X7B, draft_layers=1, draft_inter=14336)
ar_steps = iters * (k + 1) + 1
eng = VerifyEngine(shape, max_batch=b, max_verify=k + 1, max_seq=prompt + ar_steps + iters * (k + 1) + 64,
                   compress_experts=True)
rng = np.random.default_rng(2508)
prompts = rng.integers(0, shape.vocab, size=(b, prompt)).astype(np.int32)
stream = torch.cuda.Stream()
sh = stream.cuda_stream

# 1. plain greedy decoding (k = 0): the continuation + its committed tokens/s
eng.prefill(prompts, stream=sh)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(stream)
for _ in range(ar_steps):
    eng.decode_step(0, stream=sh)
e1.record(stream)
stream.synchronize()
t_ar = e0.elapsed_time(e1) * 1e-3
greedy, n_ar, _, _ = eng.decode_read(b, ar_steps)
assert np.all(n_ar == ar_steps)

# 2. same prompts, planted drafts with chain acceptance p
eng.prefill(prompts, stream=sh)
pos = np.zeros(b, np.int64)
committed, t_spec = 0, 0.0
agree, total_new = 0, 0  # bf16 near-ties between the k=8 and k=0 passes can flip a greedy token
acc_hist = []
for it in range(iters):
    drafts = np.zeros((b, k), np.int32)
    for r in range(b):
        cut = 0
        while cut < k and rng.random() < p:
            cut += 1
        cont = greedy[r, pos[r]:pos[r] + k]
        drafts[r] = cont
        drafts[r, cut:] = (cont[cut:] + 1 + np.arange(k - cut)) % shape.vocab
    stream.synchronize()
    e0.record(stream)
    eng.decode_step(k, drafts, stream=sh)
    e1.record(stream)
    stream.synchronize()
    t_spec += e0.elapsed_time(e1) * 1e-3
    com, n, _, _ = eng.decode_read(b, ar_steps)
    for r in range(b):
        new = com[r, pos[r]:n[r]]
        agree += int(np.sum(new == greedy[r, pos[r]:n[r]]))
        total_new += len(new)
        acc_hist.append(len(new) - 1)
    committed += int((n - pos).sum())
    pos = n.astype(np.int64)

alpha = float(np.mean(acc_hist)) + 1.0
out = {"workload": "mixtral-8x7b offloaded decode, b=32, prompt 1024, coded expert transfer",
       "plain_greedy": {"committed_tokens_per_s": b * ar_steps / t_ar, "ms_per_iteration": t_ar / ar_steps * 1e3},
       "speculative_k8_p0.8": {"committed_tokens_per_s": committed / t_spec, "ms_per_iteration": t_spec / iters * 1e3,
                               "mean_committed_per_request_iteration": alpha,
                               "reference_alpha_k8_p0.8": sum(p ** i for i in range(k + 1))},
       "speedup": (committed / t_spec) / (b * ar_steps / t_ar),
       "greedy_agreement": agree / max(1, total_new), "iterations": iters}
print(json.dumps(out))
eng.close()
