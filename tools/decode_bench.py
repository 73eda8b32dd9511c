"""Decode-loop launch overhead: eager iterations vs one CUDA graph per
iteration on a small model where the host, not the link, is the limit
(BASELINE config 1 shape, experts in pinned host DRAM). Prints JSON lines."""
import dataclasses
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_21706_b200 import _lib  # noqa: E402
from paper_2508_21706_b200.engine import TINY, VerifyEngine  # noqa: E402

b, k, iters = 4, 4, 40
shape = dataclasses.replace(TINY, draft_layers=1, draft_inter=512)
prompts = np.random.default_rng(0).integers(0, shape.vocab, size=(b, 256)).astype(np.int32)
stream = torch.cuda.Stream()
for graph in (False, True):
    eng = VerifyEngine(shape, max_batch=b, max_verify=k + 1, max_seq=256 + 2 * (iters + 8) * (k + 1) + 64)
    eng.prefill(prompts)
    eng.decode_run(k, 3, graph=graph, stream=stream.cuda_stream)  # warm-up (+ capture)
    stream.synchronize()
    l0 = _lib.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(stream)
    eng.decode_run(k, iters, graph=graph, stream=stream.cuda_stream)
    e1.record(stream)
    t_host = time.perf_counter() - t0
    stream.synchronize()
    t = e0.elapsed_time(e1) * 1e-3
    _, n, _, _ = eng.decode_read(b, 1)
    print(json.dumps({"mode": "cuda graph" if graph else "eager", "iterations": iters, "k": k, "batch": b,
                      "ms_per_iteration": t / iters * 1e3, "host_enqueue_ms_per_iteration": t_host / iters * 1e3,
                      "kernel_launches_per_iteration": (_lib.launch_count() - l0) / iters,
                      "verified_tokens_per_s": b * (k + 1) * iters / t}))
    eng.close()
