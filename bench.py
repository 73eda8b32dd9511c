#!/usr/bin/env python
"""Benchmark: the offloaded speculative verify step (BASELINE.json config 2).

Workload (N=1): Mixtral-8x7B shape (h 4096, h_i 14336, 8 experts top-2, 32
layers, 32/8 heads x 128, vocab 32000), bf16 procedural random-init weights,
all 90.2 GB of experts in pinned host DRAM and streamed to HBM every step
(hot-expert cache 0 by default), batch 32, draft length k (default 8 -> 9
verify rows per request), KV prefix 1024 per request. One step = one verify
pass over the batch: 32 layers of RMSNorm/QKV/RoPE/K1 attention/O/router/
permute/SwiGLU experts/combine, LM head + fused argmax, greedy accept.

Metric: verified decode tokens/s = b*(k+1)*steps / time (whole job, max over
ranks). `value` times the device-resident-input path (CUDA events on the
launch stream); `e2e` goes through the public engine API with host token
buffers (H2D of inputs + D2H of the accept result inside the timed region).

`--impl reference` runs the reference's CPU path instead (see cpu_reference()).
Under torchrun N>1 the ranks run expert parallelism: rank r
owns experts e % N == r and streams only those; the global batch is split
over the ranks (strong scaling). Setup failures abort (no replica fallback).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
H2D_FALLBACK_GBS = 55.5  # pinned H2D measured on this pool's B200 boxes (tools/probe_box.py)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--k", type=int, default=8, help="draft length (verify rows = k+1)")
    ap.add_argument("--prefix", type=int, default=1024)
    ap.add_argument("--model", default="mixtral-8x7b",
                    choices=["mixtral-8x7b", "tiny", "mixtral-8x22b", "dsv2-lite", "qwen2-57b"])
    ap.add_argument("--cache-gb", type=float, default=0.0, help="hot-expert HBM cache (GB)")
    ap.add_argument("--alias", type=int, default=0, help="host_alias_layers (0 = one pinned buffer per layer)")
    ap.add_argument("--slots", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-decode", action="store_true", help="skip the prefill + decode-loop measurement")
    ap.add_argument("--moe-batching", default="large", choices=["large", "one"],
                    help="LARGE_BATCH (stream whole layers ahead) or BATCH_ONE (stream router-selected experts)")
    ap.add_argument("--no-compress", dest="compress", action="store_false",
                    help="stream raw bf16 experts instead of the lossless code (default: coded, expanded in HBM)")
    ap.add_argument("--codec", default="auto", choices=["auto", "unary", "tile", "tile3"],
                    help="link code of the coded transfer: auto (the engine probes the first expert block: T3 "
                         "when the hot cache holds every block, else the smaller of unary and T2 — unary for "
                         "uniform-init, T2 for gaussian-like weights), unary (xfer.cu; blocks expanded in HBM by a "
                         "decode kernel), tile (tcode.cuh T2) or tile3 (T3, fixed 3-bit exponents; both decoded "
                         "inside the expert kernel, no bf16 expert in HBM)")
    ap.add_argument("--ep-transport", default="ipc", choices=["ipc", "nccl"],
                    help="N>1 expert-parallel exchange: CUDA-IPC peer mailboxes written by the dispatch / "
                         "combine kernels themselves (default; falls back to NCCL if IPC cannot be set up) "
                         "or NCCL grouped send/recv (the library baseline)")
    ap.add_argument("--init", default="uniform", choices=["uniform", "gaussian"],
                    help="routed-expert weight distribution: uniform (default, the survey's procedural init) or "
                         "gaussian-like trained weights with 1/1024 outliers (same variance); changes only the "
                         "link code's compression ratio")
    ap.add_argument("--no-raw", dest="raw", action="store_false",
                    help="skip the second timed loop with raw bf16 streaming (raw_value)")
    ap.add_argument("--micro-batches", type=int, default=1,
                    help="Hyperparameters.m: the batch as m micro-batches, stage-major per layer "
                         "(pipeline.hpp:147-206); with --attn-cpu the host attends one while the GPU runs the next")
    ap.add_argument("--attn-cpu", action="store_true",
                    help="AttentionPlacement::CPU: target K/V in pinned host DRAM, attention on the host pool")
    return ap.parse_args()


def shape_of(name):
    from paper_2508_21706_b200 import engine as E
    return {"mixtral-8x7b": E.MIXTRAL_8X7B, "tiny": E.TINY, "mixtral-8x22b": E.MIXTRAL_8X22B,
            "dsv2-lite": E.DSV2_LITE, "qwen2-57b": E.QWEN2_57B}[name]


def peaks():
    try:
        with open(PEAKS) as f:
            p = json.load(f)
        return p, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            time.sleep(0.6)  # let nvidia-smi start sampling before the timed region
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, smax, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                smax = max(smax, float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(names, f[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": smax or None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------- dist
def dist_init():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        import torch
        if SHARE_DEVICE:  # all ranks on cuda:0 (validates the N > 1 path on a 1-GPU box; NCCL refuses)
            local = 0
            torch.cuda.set_device(0)
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    return world, rank, local


# SMO_SHARE_DEVICE=1: every rank uses cuda:0 with gloo plumbing and the
# peer-memory (IPC) transport — a functional check of the expert-parallel
# bench path on one GPU, not a scaling measurement
SHARE_DEVICE = os.environ.get("SMO_SHARE_DEVICE", "0") == "1"


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(world, v):
    if world == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device="cpu" if SHARE_DEVICE else "cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ---------------------------------------------------------------- CPU path
class CpuLayerSample:
    """One verify layer of the workload on the host CPU + the LM head on a row
    sample. Attention: the reference's own moeplan::chunked_attention (fp64,
    unmodified, oracle/_ref/libmoeplan_ref_fast.so) over all b x n_q
    (request, head) instances on `threads` std::threads — the paper's CPU
    attention placement. Stages the reference does not implement (dense
    projections, router, permute, SwiGLU experts, combine, LM head) run on the
    oracle's C port (oracle/liboracle.so, OpenMP). Weights are generated once;
    run() returns (extrapolated step seconds, layer seconds, stage seconds)."""

    def __init__(self, shape, b, n, prefix, threads, use_reference=True):
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        os.environ.setdefault("OMP_NUM_THREADS", str(threads))
        import ctypes as C
        import oracle_py as O
        O.build()
        self.O, self.L = O, O.lib()
        s = self.s = shape
        self.b, self.n, self.prefix, self.threads, self.use_reference = b, n, prefix, threads, use_reference
        T = b * n
        h, hi, E = s.hidden, s.inter, s.n_expert
        nq, nkv, d = s.n_q_heads, s.n_kv_heads, s.head_dim
        self.s_max = s_max = prefix + n
        rng = np.random.default_rng(0)
        self.x = rng.uniform(-1, 1, size=(T, h)).astype(np.float32)
        self.ones = np.full(h, 0x3F80, np.uint16)
        self.wqkv = O.fill_uniform_bf16((nq + 2 * nkv) * d * h, s.seed, 1001, float(np.sqrt(3 / h)))
        self.wo = O.fill_uniform_bf16(h * nq * d, s.seed, 1002, float(np.sqrt(3 / (nq * d))))
        self.wr = O.fill_uniform_bf16(E * h, s.seed, 1004, float(np.sqrt(3 / h)))
        self.experts = [[O.fill_uniform_bf16(hi * h, s.seed, 1100 + 3 * e + j, float(np.sqrt(3 / h)))
                         for j in range(3)] for e in range(E)]
        self.kc = O.fill_uniform_bf16(b * nkv * s_max * d, s.seed, 900000, 1.0).reshape(b, nkv, s_max, d)
        self.vc = O.fill_uniform_bf16(b * nkv * s_max * d, s.seed, 900001, 1.0).reshape(b, nkv, s_max, d)
        self.mask = np.array([(1 << (i + 1)) - 1 for i in range(n)] * b, np.uint64)
        self.pre = np.full(b, prefix, np.int32)
        self.lm_rows = 8
        self.lm = O.fill_uniform_bf16(s.vocab * h, s.seed, 2, float(np.sqrt(3 / h)))
        self.shared = None
        if getattr(s, "shared_inter", 0):
            si = s.shared_inter
            self.shared = [O.fill_uniform_bf16(si * h, s.seed, 1050 + j, float(np.sqrt(3 / (h if j < 2 else si))))
                           for j in range(3)]
        if use_reference:
            R = C.CDLL(os.path.join(ROOT, "oracle", "_ref", "libmoeplan_ref_fast.so"))
            R.ref_verify_layer_attention.restype = C.c_double
            R.ref_verify_layer_attention.argtypes = [C.c_void_p] * 5 + [C.c_int] * 7 + [C.c_void_p]
            self.R = R

    def run(self):
        O, L, s = self.O, self.L, self.s
        b, n, prefix, threads = self.b, self.n, self.prefix, self.threads
        T = b * n
        h, hi, E, k = s.hidden, s.inter, s.n_expert, s.top_k
        nq, nkv, d = s.n_q_heads, s.n_kv_heads, s.head_dim
        s_max = self.s_max
        P = O._ptr
        x, ones = self.x, self.ones
        t = {}
        t0 = time.perf_counter()
        xn = np.zeros((T, h), np.uint16)
        L.orc_rmsnorm(P(x), P(ones), T, h, s.rms_eps, P(xn))
        qkv = np.zeros((T, (nq + 2 * nkv) * d), np.float32)
        L.orc_gemm_xwt(P(xn), P(self.wqkv), T, (nq + 2 * nkv) * d, h, P(qkv))
        qkv_b = O.f32_to_bf16(qkv)
        q = np.ascontiguousarray(qkv_b[:, :nq * d])
        pos = np.tile(prefix + np.arange(n, dtype=np.int32), b)
        L.orc_rope(P(q), T, nq, d, P(pos), s.rope_theta)
        t["pre_attn"] = time.perf_counter() - t0
        out = np.zeros((T, nq, d))
        if self.use_reference:
            ta = self.R.ref_verify_layer_attention(P(q), P(self.kc), P(self.vc), P(self.mask), P(self.pre), b, n,
                                                   nq, nkv, d, s_max, threads, P(out))
            if ta < 0:
                raise RuntimeError("reference attention failed")
            attn = O.f32_to_bf16(out.astype(np.float32))
        else:
            attn = np.zeros((T, nq, d), np.uint16)
            t1 = time.perf_counter()
            L.orc_verify_attention(P(q), P(self.kc), P(self.vc), P(self.mask), P(self.pre), b, n, nq, nkv, d,
                                   s_max, P(attn))
            ta = time.perf_counter() - t1
        t["attention"] = ta
        t0 = time.perf_counter()
        o = np.zeros((T, h), np.float32)
        L.orc_gemm_xwt(P(attn), P(self.wo), T, h, nq * d, P(o))
        x2 = x + o
        L.orc_rmsnorm(P(x2), P(ones), T, h, s.rms_eps, P(xn))
        lg = np.zeros((T, E), np.float32)
        L.orc_router_logits(P(xn), P(self.wr), T, h, E, P(lg))
        ids = np.zeros((T, k), np.int32)
        wts = np.zeros((T, k), np.float32)
        L.orc_topk_softmax(P(lg), T, E, k, P(ids), P(wts))
        t["dense_router"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        y = np.zeros((T, h), np.float64)
        for e in range(E):
            rows, slots = np.nonzero(ids == e)
            if rows.size == 0:
                continue
            X = np.ascontiguousarray(xn[rows])
            Y = np.zeros((rows.size, h), np.float32)
            w1, w3, w2 = self.experts[e]
            L.orc_expert_swiglu(P(X), rows.size, h, hi, P(w1), P(w3), P(w2), P(Y))
            y[rows] += wts[rows, slots][:, None] * Y
        if self.shared is not None:
            Ysh = np.zeros((T, h), np.float32)
            ws = self.shared
            L.orc_expert_swiglu(P(np.ascontiguousarray(xn)), T, h, s.shared_inter, P(ws[0]), P(ws[1]), P(ws[2]),
                                P(Ysh))
            y += Ysh
        t["moe"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        lr = self.lm_rows
        lo = np.zeros((lr, s.vocab), np.float32)
        L.orc_gemm_xwt(P(np.ascontiguousarray(xn[:lr])), P(self.lm), lr, s.vocab, h, P(lo))
        t["lm_head_sample"] = time.perf_counter() - t0
        layer = t["pre_attn"] + t["attention"] + t["dense_router"] + t["moe"]
        step = s.n_layers * layer + t["lm_head_sample"] * (T / lr)
        return step, layer, t


def cpu_layer_sample(shape, b, n, prefix, threads, use_reference=True):
    return CpuLayerSample(shape, b, n, prefix, threads, use_reference).run()


def cpu_baseline(shape, b, n, prefix, metric_unit):
    threads = os.cpu_count() or 1
    step, layer, parts = CpuLayerSample(shape, b, n, prefix, threads).run()
    return {"value": b * n / step, "unit": metric_unit, "cores": threads, "kind": "reference",
            "sample": (f"1 of {shape.n_layers} verify layers (b={b}, n={n}, s={prefix}) + LM head on 8 of {b * n} "
                       f"rows, extrapolated to one step ({step:.1f} s/step); attention = the reference's "
                       f"moeplan::chunked_attention (fp64, {b * shape.n_q_heads} instances, {threads} threads), "
                       f"other stages = oracle C port (the reference has no kernels for them)"),
            "stage_seconds": {k: round(v, 4) for k, v in parts.items()}}


def run_reference(args):
    """The reference's CPU path on the host cores. One step of this arm is a
    BOUNDED SAMPLE of the verify step: one of the L layers (the reference's
    own chunked_attention over every (request, head) + the oracle port for
    the stages the reference has no code for) plus the LM head on 8 rows;
    `ms_per_step` is that sample's measured time (so ms_per_step x steps is
    this run's wall time), and `value` extrapolates it to whole verify steps
    (L layers + the full LM head) — `extrapolated` says so."""
    rank = int(os.environ.get("RANK", "0"))
    shape = shape_of(args.model)
    b, n = args.batch, args.k + 1
    metric = "verified decode tokens/s"
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    cpu = CpuLayerSample(shape, b, n, args.prefix, threads)
    for _ in range(max(0, args.warmup)):
        cpu.run()
    steps, samples = [], []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        st, _, parts = cpu.run()
        samples.append(time.perf_counter() - t0)
        steps.append(st)
    t_step = float(np.mean(steps))
    t_sample = float(np.mean(samples))
    v = b * n / t_step
    line = {"impl": "reference", "metric": metric, "value": v, "unit": "tokens/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_sample * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64 attention / f32-f64 port", "data": "synthetic",
            "extrapolated": True,
            "extrapolation": {"sample": f"1 of {shape.n_layers} verify layers + LM head on 8 of {b * n} rows",
                              "sample_ms": t_sample * 1e3, "full_step_ms": t_step * 1e3,
                              "value_from": "b*(k+1) / full_step_ms",
                              "stage_seconds_last_sample": {k: round(x, 4) for k, x in parts.items()}},
            "config": {"workload": f"{args.model} verify step, b={b}, k={args.k}, s={args.prefix}, CPU host",
                       "batch": b, "draft_len": args.k, "prefix": args.prefix},
            "cpu_baseline": {"value": v, "unit": "tokens/s", "cores": threads, "kind": "reference",
                             "sample": "each step = 1 verify layer + LM-head row sample, extrapolated x"
                                       f"{shape.n_layers} layers; attention = the reference's chunked_attention "
                                       "(fp64, unmodified); dense/router/experts/LM head = the oracle's C port "
                                       "(the reference has no code for them)"},
            "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def codec_traffic_per_block(kernel="K5_expert_decode_unary"):
    """dram__bytes_read+write of one expert_decode launch (one Mixtral expert
    block) from the newest committed ncu capture (profiles/r02e_traffic.json:
    the unary decoder the engine uses; r01f_traffic.json: the 3-bit one)."""
    for f in ("r02e_traffic.json", "r01k_traffic.json", "r01j_traffic.json", "r01i_traffic.json", "r01h_traffic.json", "r01f_traffic.json"):
        try:
            k = json.load(open(os.path.join(ROOT, "profiles", f)))["kernels"][kernel]
            return k["dram_read_bytes"] + k["dram_write_bytes"]
        except Exception:
            continue
    return None


def moe_traffic_per_layer():
    """dram__bytes_read+write of one layer's expert block (the fused K4-MoE
    launch) from the committed ncu --set full capture of the bench step
    (profiles/r01c_traffic.json)."""
    p = os.path.join(ROOT, "profiles", "r01c_traffic.json")
    try:
        k = json.load(open(p))["kernels"]["K4_moe_fused"]
        return k["dram_read_bytes"] + k["dram_write_bytes"]
    except Exception:
        return None


def decode_loop(eng, shape, b, prefix, k, stream, sh, iters=3):
    """SURVEY.md §8 f1/f2 on the bench engine: layer-major prefill of b
    random prompts of `prefix` tokens (each layer's experts streamed once),
    then `iters` draft -> verify -> accept -> commit iterations with the
    on-device drafter. Random-init drafter and target: acceptance ~0, so a
    step commits ~1 token per request (the bonus); the numbers show the
    prefill throughput and the drafter's share of an iteration."""
    import torch
    rng = np.random.default_rng(77)
    prompts = rng.integers(0, shape.vocab, size=(b, prefix)).astype(np.int32)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    eng.prefill(prompts, stream=sh)
    t_pf = time.perf_counter() - t0
    pf_h2d = eng.last_times()["h2d_bytes"]
    eng.decode_step(k, stream=sh)  # warm the drafter path
    stream.synchronize()
    _, n0, _, _ = eng.decode_read(b, 1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    draft = 0.0
    e0.record(stream)
    for _ in range(iters):
        eng.decode_step(k, stream=sh)
    e1.record(stream)
    stream.synchronize()
    draft = eng.last_times()["draft"]
    t = e0.elapsed_time(e1) * 1e-3
    _, n1, kv, _ = eng.decode_read(b, 1)
    committed = int((n1 - n0).sum())
    return {"prefill": {"requests": b, "prompt_tokens": prefix, "seconds": t_pf,
                        "tokens_per_s": b * prefix / t_pf, "h2d_gbs": pf_h2d / t_pf / 1e9,
                        "note": "wall clock incl. scratch allocation; experts streamed once per layer"},
            "decode": {"k": k, "iterations": iters, "ms_per_iteration": t / iters * 1e3,
                       "verified_tokens_per_s": b * (k + 1) * iters / t, "committed_tokens_per_s": committed / t,
                       "mean_accepted_drafts": committed / (b * iters) - 1.0,
                       "draft_ms_last_iteration": draft * 1e3,
                       "drafter": f"{shape.draft_layers} dense layer(s), SwiGLU {shape.draft_inter}, random-init"}}


# ---------------------------------------------------------------- GPU path
def raw_pass(shape, args, b, n, prefix, s_max, local, h2d_peak, pk, alias=8):
    """The same verify step with raw bf16 expert streaming (no link code):
    device-timed like `value`, min(steps, 5) steps after 2 warm-up steps."""
    import torch
    from paper_2508_21706_b200.engine import VerifyEngine, step_roofline
    eng = VerifyEngine(shape, max_batch=b, max_verify=n, max_seq=s_max, hbm_slots=args.slots,
                       expert_cache_bytes=int(args.cache_gb * 1e9), host_alias_layers=alias, device=local,
                       attn_cpu=args.attn_cpu, batch_one=args.moe_batching == "one", compress_experts=False,
                       micro_batches=args.micro_batches)
    dev = torch.device(f"cuda:{local}")
    pre = np.full(b, prefix, np.int32)
    eng.fill_prefix(pre)
    tokens = torch.from_numpy(np.random.default_rng(1234).integers(0, shape.vocab, size=(b, n)).astype(np.int32)).to(dev)
    pre_d = torch.from_numpy(pre).to(dev)
    acc = torch.empty(b, dtype=torch.int32, device=dev)
    bonus = torch.empty(b, dtype=torch.int32, device=dev)
    stream = torch.cuda.Stream(device=dev)
    steps = max(1, min(args.steps, 5))
    with torch.cuda.stream(stream):
        for _ in range(2):
            eng.verify_device(tokens, pre_d, acc, bonus, stream=stream.cuda_stream)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            eng.verify_device(tokens, pre_d, acc, bonus, stream=stream.cuda_stream)
        e1.record(stream)
    stream.synchronize()
    t = e0.elapsed_time(e1) * 1e-3 / steps
    st = eng.last_times()
    roof = step_roofline(shape, b, n, prefix, h2d_peak, pk["hbm_gbs"], pk.get("bf16_tflops_sustained", 1400.0),
                         cached_blocks=int(args.cache_gb * 1e9) // shape.expert_bytes,
                         h2d_bytes=st["h2d_bytes"] if args.moe_batching == "one" else None)
    eng.close()
    return {"value": b * n / t, "unit": "tokens/s", "ms_per_step": t * 1e3, "steps": steps, "warmup": 2,
            "expert_transfer": "raw bf16", "h2d_bytes_per_step": st["h2d_bytes"],
            "h2d_gbs": st["h2d_bytes"] / t / 1e9, "step_roofline_frac": roof["t_roof_s"] / t,
            "host_alias_layers": alias}


def run_ours(args):
    import torch
    from paper_2508_21706_b200 import _lib
    from paper_2508_21706_b200.engine import VerifyEngine, geometric_alpha, step_roofline
    world, rank, local = dist_init()
    dev = torch.device(f"cuda:{local}")
    torch.cuda.set_device(dev)
    shape = shape_of(args.model)
    if args.init == "gaussian":
        import dataclasses
        shape = dataclasses.replace(shape, expert_init=_lib.INIT_GAUSSIAN)
    if world == 1 and not args.no_decode:
        # the drafter of the reference's config (DraftModelSpec, mixtral8x7b.json:
        # 1 layer, ffn_ops_per_token 3.52e8 = 6*h*draft_inter) for the decode loop
        import dataclasses
        shape = dataclasses.replace(shape, draft_layers=1,
                                    draft_inter=max(128, int(round(3.52e8 / (6 * shape.hidden) / 128)) * 128))
    b, n, prefix = args.batch, args.k + 1, args.prefix
    pk, pk_kind = peaks()
    s_max = prefix + n + 64
    t_create = time.perf_counter()
    alias = args.alias
    # N > 1: expert parallelism over NCCL: rank r owns experts
    # e % N == r and streams only that shard; the global batch b is split over
    # the ranks (attention is data-parallel over requests) -> strong scaling.
    mode, grp = "1 GPU", None
    ep_rank, ep_size = 0, 1
    if world > 1:
        from paper_2508_21706_b200.engine import EpGroup
        import torch.distributed as dist
        gloo = dist.new_group(backend="gloo")  # host barriers of the peer-memory transport (collective call)
        try:
            if b % world or shape.n_expert % world:
                raise ValueError(f"batch {b} / experts {shape.n_expert} not divisible by {world}")
            grp = None

            def make_nccl():
                uid = [EpGroup.nccl_unique_id() if rank == 0 else None]
                dist.broadcast_object_list(uid, src=0)
                return EpGroup.nccl(uid[0], world, rank)

            def make_ipc():  # peer mailboxes over NVLink, stored into by the EP kernels, no NCCL
                def all_gather(blob):
                    out = [None] * world
                    dist.all_gather_object(out, blob, group=gloo)
                    return out
                return EpGroup.ipc(world, rank, EpGroup.ipc_slot_bytes(shape, b // world, n), all_gather,
                                   lambda: dist.barrier(group=gloo))

            order = ["ipc"] if SHARE_DEVICE else ([args.ep_transport] + [t for t in ("ipc", "nccl")
                                                                          if t != args.ep_transport])
            for tname in order:
                try:
                    grp = make_ipc() if tname == "ipc" else make_nccl()
                    args.ep_transport = tname
                    break
                except Exception as ex:
                    print(f"[bench] {tname} transport unavailable ({ex})", file=sys.stderr)
            if grp is None:
                raise RuntimeError("no expert-parallel transport")
            ep_rank, ep_size, mode = rank, world, f"ep{world} ({args.ep_transport})"
            b = b // world
        except Exception as ex:  # fail loudly: a replica run would not measure the EP path
            raise RuntimeError(f"expert parallelism over {world} ranks could not be set up: {ex}") from ex
    eng = None
    if args.codec == "unary":  # pin the unary code (no probe)
        os.environ["SMO_CODEC"] = "unary"
    for a in (alias, 8, 4, 2):
        try:
            eng = VerifyEngine(shape, max_batch=b, max_verify=n, max_seq=s_max, hbm_slots=args.slots,
                               expert_cache_bytes=int(args.cache_gb * 1e9), host_alias_layers=a, device=local,
                               ep_rank=ep_rank, ep_size=ep_size, ep_group=grp, attn_cpu=args.attn_cpu,
                               batch_one=args.moe_batching == "one",
                               compress_experts=({"tile": 2, "tile3": 3}.get(args.codec, 1)) if args.compress else 0,
                               micro_batches=args.micro_batches)
            alias = a
            break
        except _lib.CapacityError as e:
            print(f"[bench] engine capacity ({e}); retrying with host_alias_layers={a}", file=sys.stderr)
    t_create = time.perf_counter() - t_create
    prefix_arr = np.full(b, prefix, np.int32)
    eng.fill_prefix(prefix_arr)
    rng = np.random.default_rng(1234 + rank)
    tokens_h = rng.integers(0, shape.vocab, size=(b, n)).astype(np.int32)
    tokens = torch.from_numpy(tokens_h).to(dev)
    pre_d = torch.from_numpy(prefix_arr).to(dev)
    acc = torch.empty(b, dtype=torch.int32, device=dev)
    bonus = torch.empty(b, dtype=torch.int32, device=dev)
    stream = torch.cuda.Stream(device=dev)
    sh = stream.cuda_stream

    # live H2D link peak on this box (pinned, 2 GiB copies)
    hbuf = torch.empty(1 << 31, dtype=torch.uint8, pin_memory=True)
    dbuf = torch.empty(1 << 31, dtype=torch.uint8, device=dev)
    h2d_peak = 0.0
    with torch.cuda.stream(stream):
        dbuf.copy_(hbuf, non_blocking=True)
        for _ in range(4):  # best of four 2 GiB copies
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            dbuf.copy_(hbuf, non_blocking=True)
            e1.record(stream)
            stream.synchronize()
            h2d_peak = max(h2d_peak, (1 << 31) / (e0.elapsed_time(e1) * 1e-3) / 1e9)
    del hbuf, dbuf
    torch.cuda.empty_cache()

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            eng.verify_device(tokens, pre_d, acc, bonus, stream=sh)
    stream.synchronize()
    barrier(world)
    torch.cuda.synchronize()
    l0 = _lib.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    prof = os.environ.get("SMO_PROFILE_TIMED") == "1"  # ncu --profile-from-start off: the timed steps only
    with ClockSampler(local) as clk:
        if prof:
            torch.cuda.cudart().cudaProfilerStart()
        with torch.cuda.stream(stream):
            ev0.record(stream)
            for _ in range(args.steps):
                eng.verify_device(tokens, pre_d, acc, bonus, stream=sh)
            ev1.record(stream)
        stream.synchronize()
        if prof:
            torch.cuda.cudart().cudaProfilerStop()
    launches = _lib.launch_count() - l0
    t_local = ev0.elapsed_time(ev1) * 1e-3
    barrier(world)
    t_all = max_over_ranks(world, t_local)
    stages = eng.last_times()  # per-stage durations of the last timed step
    verified = world * b * n * args.steps
    value = verified / t_all
    ms_step = t_all / args.steps * 1e3

    # e2e through the public API with host buffers (pinned staging inside)
    e2e = None
    if not args.no_e2e:
        for _ in range(1):
            eng.verify(tokens_h, prefix_arr, stream=sh)
        barrier(world)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            res = eng.verify(tokens_h, prefix_arr, stream=sh)
        t_e2e = max_over_ranks(world, time.perf_counter() - t0)
        e2e = {"value": world * b * n * args.steps / t_e2e, "unit": "tokens/s",
               "h2d_bytes_per_step": int(tokens_h.nbytes + prefix_arr.nbytes),
               "d2h_bytes_per_step": int(res.acc_len.nbytes + res.bonus.nbytes + res.keep.nbytes +
                                         res.target.nbytes),
               "api": "smo_engine_verify (host buffers)"}

    decode = None
    if world == 1 and not args.no_decode:
        try:
            decode = decode_loop(eng, shape, b, prefix, args.k, stream, sh)
        except Exception as ex:  # reported, never hides the headline
            decode = {"error": str(ex)}

    cached = int(args.cache_gb * 1e9) // shape.expert_bytes
    codec_hbm = float(stages.get("codec_bytes") or 0.0)  # code read + bf16 written by the block expansion
    # (1) against SURVEY.md §8(d)'s algorithmic bytes: the bf16 expert blocks
    # (roofline.hpp:61-62; BATCH_ONE: the routed ones) — the codec can beat it
    roof_alg = step_roofline(shape, b * ep_size, n, prefix, h2d_peak, pk["hbm_gbs"],
                             pk.get("bf16_tflops_sustained", 1400.0), cached_blocks=cached, ep=ep_size,
                             h2d_bytes=stages["h2d_raw_bytes"] if args.moe_batching == "one" else None,
                             extra_hbm_bytes=codec_hbm)
    # (2) against the bytes that actually crossed the link (coded blocks)
    roof = step_roofline(shape, b * ep_size, n, prefix, h2d_peak, pk["hbm_gbs"],
                         pk.get("bf16_tflops_sustained", 1400.0), cached_blocks=cached, ep=ep_size,
                         h2d_bytes=stages["h2d_bytes"] if (args.moe_batching == "one" or args.compress) else None,
                         extra_hbm_bytes=codec_hbm)
    h2d_bytes = stages["h2d_bytes"]
    t_step = t_all / args.steps
    raw_h2d = stages["h2d_raw_bytes"]  # the bf16 bytes those transfers carry (coded blocks expand)
    # dominant GPU kernel by device time: K4 grouped SwiGLU (+down +combine),
    # HBM-bound: algorithmic bytes = expert weights read once per layer
    moe_bytes_step = shape.n_layers * (shape.n_expert // ep_size) * shape.expert_bytes
    if args.moe_batching == "one":  # only routed experts are read: the streamed ones + the hot cache
        moe_bytes_step = stages["h2d_raw_bytes"] + int(args.cache_gb * 1e9) // shape.expert_bytes * shape.expert_bytes
    moe_t = stages["gpu_moe"]
    attn_bytes_step = shape.n_layers * 2 * b * (prefix + n) * shape.n_kv_heads * shape.head_dim * 2
    # the fused expert kernel (per step: expert bytes / kernel time from CUDA events on its stream)
    moe_roof = {"bound": "hbm", "kernel": "K4-MoE fused expert block (gate/up + SwiGLU + down, one persistent launch "
                "per layer; CUDA events around the launch on its stream), per step",
                "achieved": moe_bytes_step / moe_t / 1e9 if moe_t > 0 else None, "peak": pk["hbm_gbs"],
                "unit": "GB/s", "frac": (moe_bytes_step / moe_t / 1e9) / pk["hbm_gbs"] if moe_t > 0 else None,
                "traffic": moe_traffic_per_layer() if (args.model == "mixtral-8x7b" and ep_size == 1
                                                       and stages.get("link_code", 0) < 2) else None,
                "traffic_unit": "dram bytes per layer (the fused expert launch, ncu profiles/r01c_traffic.json); "
                "algorithmic per layer = " + str((shape.n_expert // ep_size) * shape.expert_bytes),
                "peak_kind": pk_kind}
    # with the coded transfer the block expansion is the largest device-time kernel
    # (profiles/r01h_launches.md): algorithmic bytes = code read + bf16 written
    codec_roof = None
    if args.compress and stages.get("codec", 0) > 0:
        cb = stages.get("codec_bytes") or (stages["h2d_bytes"] + stages["h2d_raw_bytes"])
        codec_roof = {"bound": "hbm", "kernel": "K5 expert_decode (coded blocks -> bf16 HBM slot), per step",
                      "achieved": cb / stages["codec"] / 1e9, "peak": pk["hbm_gbs"], "unit": "GB/s",
                      "frac": cb / stages["codec"] / 1e9 / pk["hbm_gbs"], "traffic": codec_traffic_per_block(),
                      "traffic_unit": "dram bytes per expert block (one layer's decode launch / its blocks, ncu "
                      "profiles/r02e_traffic.json); algorithmic per block = "
                      + str(int((stages["code_bits"] / 16.0 + 1.0) * shape.expert_bytes)),
                      "bound_note": "the unary decoder is integer-pipe bound (ALU pipe 81 % of peak, issue slots "
                      "78 % busy, ncu profiles/r02e_unary_decode.md); HBM is not its limiter",
                      "peak_kind": pk_kind}
    line = {
        "metric": "verified decode tokens/s", "value": value, "unit": "tokens/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong" if ep_size > 1 else "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (procedural random-init)",
        "config": {"workload": f"{args.model} offloaded verify step (BASELINE config "
                   f"{ {'mixtral-8x7b': 2, 'dsv2-lite': 4, 'qwen2-57b': 4, 'mixtral-8x22b': 5}.get(args.model, 1)})", "batch": b * ep_size,
                   "draft_len": args.k, "verify_rows": b * n, "prefix": prefix, "experts_in": "pinned host DRAM",
                   "expert_cache_gb": args.cache_gb, "hbm_slots": args.slots, "host_alias_layers": alias,
                   "attention_placement": "CPU (host K/V, host thread pool)" if args.attn_cpu else "GPU_RESIDENT (K1)",
                   "micro_batches": args.micro_batches,
                   "moe_batching": "BATCH_ONE (router-selected experts)" if args.moe_batching == "one"
                   else "LARGE_BATCH (whole layers)",
                   "expert_transfer": (f"lossless tile-coded blocks (tcode.cuh T{int(stages['link_code'])}, "
                                       f"{stages['code_bits']:.2f} "
                                       "bits/weight), decoded in shared memory by the expert kernel"
                                       if stages.get("link_code", 0) >= 2 else
                                       f"lossless exponent-coded blocks (xfer.cu, "
                                       f"{stages['code_bits']:.2f} "
                                       "bits/weight), expanded in HBM before the expert kernel")
                   if args.compress else "raw bf16",
                   "l2": "inputs larger than L2 (90.2 GB of experts + 4.6 GB KV streamed per step)",
                   "expert_init": args.init,
                   "host_numa_node": int(stages.get("host_numa", -1)),
                   "parallelism": mode},
        "committed_tokens_per_s_model": world * b * geometric_alpha(0.8, args.k) / t_step,
        "h2d": {"achieved_gbs": h2d_bytes / t_step / 1e9, "link_peak_gbs": h2d_peak,
                "bytes_per_step": h2d_bytes, "copy_engine_busy_s": stages["h2d_transfer"],
                "raw_bf16_bytes_per_step": raw_h2d, "raw_equivalent_gbs": raw_h2d / t_step / 1e9},
        "roofline": codec_roof if codec_roof else moe_roof,
        "expert_roofline": moe_roof,
        "step_roofline": {"bound": roof_alg["bound"], "t_roof_s": roof_alg["t_roof_s"], "t_meas_s": t_step,
                          "frac": roof_alg["t_roof_s"] / t_step, "h2d_bytes": roof_alg["h2d_bytes"],
                          "hbm_bytes": roof_alg["hbm_bytes"], "times_s": roof_alg["times"],
                          "note": "SURVEY.md §8(d) algorithmic bytes (bf16 expert blocks over the link); "
                                  "frac > 1 means the lossless link code beat the bf16 link roofline",
                          "link_bytes": {"bound": roof["bound"], "t_roof_s": roof["t_roof_s"],
                                         "frac": roof["t_roof_s"] / t_step, "h2d_bytes": roof["h2d_bytes"],
                                         "times_s": roof["times"],
                                         "note": "the same rule on the bytes that actually crossed the link"},
                          "h2d_peak_gbs": h2d_peak, "hbm_peak_gbs": pk["hbm_gbs"],
                          "hbm_term_includes_codec_bytes": codec_hbm},
        "codec_bits_per_weight": stages["code_bits"],  # the blocks as stored (host + coded cache)
        "link_bits_per_weight": (16.0 * stages["h2d_bytes"] / stages["h2d_raw_bytes"]
                                 if stages["h2d_raw_bytes"] > 0 else None),  # what crossed the link this step
        "expert_tflops": (shape.n_layers * 2 * 3 * shape.hidden * shape.inter * b * n * shape.top_k / moe_t / 1e12
                          if moe_t > 0 else None),
        "attention_roofline": {"bound": "hbm", "achieved": attn_bytes_step / stages["attention"] / 1e9
                               if stages["attention"] > 0 else None, "peak": pk["hbm_gbs"], "unit": "GB/s"},
        "stage_seconds_last_step": {k: stages[k] for k in ("target_total", "attention", "gpu_moe", "codec",
                                                           "h2d_transfer", "others")},
        "gpu_launches": launches, "engine_create_s": t_create,
    }
    line["clocks"] = clk.summary()
    if world == 1 and args.compress and args.raw:
        # second timed loop, raw bf16 experts on the link (the same bytes the
        # survey's roofline counts); pinned buffers aliased over 8 layers to
        # bound host memory — every step still moves all L*E blocks
        eng.close()
        try:
            line["raw"] = raw_pass(shape, args, b, n, prefix, s_max, local, h2d_peak, pk)
            line["raw_value"] = line["raw"]["value"]
        except Exception as ex:  # reported, never hides the headline
            line["raw"] = {"error": str(ex)}
    if decode:
        line["decode_loop"] = decode
    if e2e:
        line["e2e"] = e2e
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            line["cpu_baseline"] = cpu_baseline(shape, b, n, prefix, "tokens/s")
        except Exception as ex:  # reported, never a fallback
            line["cpu_baseline"] = {"error": str(ex)}
    if rank == 0:
        print(json.dumps(line), flush=True)
    eng.close()
    if grp is not None:
        grp.close()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
