"""CPU oracle of one verify step of the procedural Mixtral-style model.

TEST INFRASTRUCTURE: composes the C restatement in oracle/liboracle.so with the
same procedural tensor ids and scales as the engine (engine.cu namespace tid,
DESIGN.md §3.1), so the oracle regenerates bit-identical weights and KV.
"""
from __future__ import annotations

import math

import numpy as np

import oracle_py as O

PHI = 0x9E3779B97F4A7C15


def tid_layer(l):
    return 1000 * (l + 1)


class OracleModel:
    def __init__(self, shape, host_alias_layers=0):
        self.s = shape
        self.alias = host_alias_layers or shape.n_layers
        s = shape
        self.qkv_w = (s.n_q_heads + 2 * s.n_kv_heads) * s.head_dim
        self.ones = np.full(s.hidden, 0x3F80, np.uint16)
        self._cache = {}

    def _fill(self, count, tid, scale, base=0):
        return O.fill_uniform_bf16(count, self.s.seed, tid, scale, base)

    def embed(self):
        s = self.s
        if "embed" not in self._cache:
            self._cache["embed"] = self._fill(s.vocab * s.hidden, 1, 1.0).reshape(s.vocab, s.hidden)
        return self._cache["embed"]

    def lm_head(self):
        s = self.s
        if "lm" not in self._cache:
            self._cache["lm"] = self._fill(s.vocab * s.hidden, 2, math.sqrt(3.0 / s.hidden) * s.lm_scale).reshape(
                s.vocab, s.hidden)
        return self._cache["lm"]

    def wqkv(self, l):
        s = self.s
        return self._fill(self.qkv_w * s.hidden, tid_layer(l) + 1, math.sqrt(3.0 / s.hidden)).reshape(
            self.qkv_w, s.hidden)

    def wo(self, l):
        s = self.s
        k = s.n_q_heads * s.head_dim
        return self._fill(s.hidden * k, tid_layer(l) + 2, math.sqrt(3.0 / k)).reshape(s.hidden, k)

    def router(self, l):
        s = self.s
        return self._fill(s.n_expert * s.hidden, tid_layer(l) + 4,
                          math.sqrt(3.0 / s.hidden) * s.router_scale).reshape(s.n_expert, s.hidden)

    def shared(self, l):
        s = self.s
        if not getattr(s, "shared_inter", 0):
            return None
        h, si = s.hidden, s.shared_inter
        base = tid_layer(l) + 50
        w1 = self._fill(si * h, base, math.sqrt(3.0 / h)).reshape(si, h)
        w3 = self._fill(si * h, base + 1, math.sqrt(3.0 / h)).reshape(si, h)
        w2 = self._fill(h * si, base + 2, math.sqrt(3.0 / si)).reshape(h, si)
        return w1, w3, w2

    def expert(self, l, e):
        s = self.s
        a = l % self.alias
        base = tid_layer(a) + 100 + 3 * e
        h, hi = s.hidden, s.inter
        fill = self._fill
        if getattr(s, "expert_init", 0) == 1:  # gaussian-like trained weights (orc_fill_normal_bf16)
            fill = lambda count, tid, scale: O.fill_normal_bf16(count, self.s.seed, tid, scale)  # noqa: E731
        w1 = fill(hi * h, base, math.sqrt(3.0 / h)).reshape(hi, h)
        w3 = fill(hi * h, base + 1, math.sqrt(3.0 / h)).reshape(hi, h)
        w2 = fill(h * hi, base + 2, math.sqrt(3.0 / hi)).reshape(h, hi)
        return w1, w3, w2

    def kv_prefix(self, l, which, prefix, s_max):
        """[b, n_kv, s_max, d] bf16 with the synthetic prefix rows filled."""
        s = self.s
        b = len(prefix)
        out = np.zeros((b, s.n_kv_heads, s_max, s.head_dim), np.uint16)
        tid = 900000 + 2 * l + which
        for r in range(b):
            for hk in range(s.n_kv_heads):
                rh = r * s.n_kv_heads + hk
                n = int(prefix[r]) * s.head_dim
                out[r, hk, :prefix[r]] = self._fill(n, tid, 1.0, base=rh << 32).reshape(prefix[r], s.head_dim)
        return out

    # ---------------------------------------------------------------- stages
    def rmsnorm(self, x):
        T, h = x.shape
        y = np.zeros((T, h), np.uint16)
        O.lib().orc_rmsnorm(O._ptr(np.ascontiguousarray(x, np.float32)), O._ptr(self.ones), T, h,
                            self.s.rms_eps, O._ptr(y))
        return y

    @staticmethod
    def gemm(X, W):
        X = np.ascontiguousarray(X, np.uint16)
        W = np.ascontiguousarray(W, np.uint16)
        T, K = X.shape
        N = W.shape[0]
        out = np.zeros((T, N), np.float32)
        O.lib().orc_gemm_xwt(O._ptr(X), O._ptr(W), T, N, K, O._ptr(out))
        return out

    def rope(self, x_bf16, positions, heads):
        x = np.ascontiguousarray(x_bf16, np.uint16).copy()
        pos = np.ascontiguousarray(positions, np.int32)
        O.lib().orc_rope(O._ptr(x), x.shape[0], heads, self.s.head_dim, O._ptr(pos), self.s.rope_theta)
        return x

    def attention(self, q, kc, vc, mask_bits, prefix, n):
        s = self.s
        b = len(prefix)
        out = np.zeros_like(q)
        rc = O.lib().orc_verify_attention(O._ptr(np.ascontiguousarray(q)), O._ptr(np.ascontiguousarray(kc)),
                                          O._ptr(np.ascontiguousarray(vc)),
                                          O._ptr(np.ascontiguousarray(mask_bits, np.uint64)),
                                          O._ptr(np.ascontiguousarray(prefix, np.int32)), b, n, s.n_q_heads,
                                          s.n_kv_heads, s.head_dim, kc.shape[2], O._ptr(out))
        assert rc == 0, rc
        return out

    def router_logits(self, xn, l):
        T = xn.shape[0]
        lg = np.zeros((T, self.s.n_expert), np.float32)
        O.lib().orc_router_logits(O._ptr(np.ascontiguousarray(xn)), O._ptr(self.router(l)), T, self.s.hidden,
                                  self.s.n_expert, O._ptr(lg))
        return lg

    def topk(self, logits):
        T, E = logits.shape
        k = self.s.top_k
        ids = np.zeros((T, k), np.int32)
        w = np.zeros((T, k), np.float32)
        O.lib().orc_topk_softmax(O._ptr(np.ascontiguousarray(logits)), T, E, k, O._ptr(ids), O._ptr(w))
        return ids, w

    def permute(self, ids):
        T, k = ids.shape
        E = self.s.n_expert
        off = np.zeros(E + 1, np.int32)
        perm = np.zeros(T * k, np.int32)
        pos = np.zeros(T * k, np.int32)
        O.lib().orc_permute(O._ptr(np.ascontiguousarray(ids)), T, k, E, O._ptr(off), O._ptr(perm), O._ptr(pos))
        return off, perm, pos

    def moe(self, xn, l, ids, w):
        """Returns y [T, h] = sum_j w_j * expert_{ids_j}(xn)."""
        s = self.s
        T = xn.shape[0]
        y = np.zeros((T, s.hidden), np.float64)
        for e in range(s.n_expert):
            rows, slots = np.nonzero(ids == e)
            if rows.size == 0:
                continue
            w1, w3, w2 = self.expert(l, e)
            X = np.ascontiguousarray(xn[rows])
            Y = np.zeros((rows.size, s.hidden), np.float32)
            O.lib().orc_expert_swiglu(O._ptr(X), rows.size, s.hidden, s.inter, O._ptr(w1), O._ptr(w3), O._ptr(w2),
                                      O._ptr(Y))
            y[rows] += w[rows, slots][:, None].astype(np.float64) * Y
        return y

    @staticmethod
    def depth(parent, n):
        if parent is None:
            return np.arange(n)
        d = np.zeros(n, np.int64)
        for i in range(1, n):
            d[i] = d[parent[i]] + 1
        return d

    @staticmethod
    def mask_bits(parent, n):
        bits = np.zeros(n, np.uint64)
        for i in range(n):
            if parent is None:
                bits[i] = (1 << (i + 1)) - 1 if i < 63 else 0xFFFFFFFFFFFFFFFF
            else:
                m, cur = 0, i
                while cur >= 0:
                    m |= 1 << cur
                    cur = -1 if cur == 0 else int(parent[cur])
                bits[i] = m
        return bits

    def layer(self, l, x, kc, vc, prefix, n, parents=None):
        """One decoder layer from fp32 residual x [T,h]; kc/vc updated in place.
        Returns (x_out, intermediates dict)."""
        s = self.s
        b = len(prefix)
        T = b * n
        xn1 = self.rmsnorm(x)
        qkv = O.f32_to_bf16(self.gemm(xn1, self.wqkv(l))).reshape(T, -1)
        d, nq, nkv = s.head_dim, s.n_q_heads, s.n_kv_heads
        q = qkv[:, :nq * d].reshape(T, nq, d)
        k = qkv[:, nq * d:(nq + nkv) * d].reshape(T, nkv, d)
        v = qkv[:, (nq + nkv) * d:].reshape(T, nkv, d)
        pos = np.zeros(T, np.int32)
        mbits = np.zeros(T, np.uint64)
        for r in range(b):
            par = None if parents is None else parents[r]
            pos[r * n:(r + 1) * n] = prefix[r] + self.depth(par, n)
            mbits[r * n:(r + 1) * n] = self.mask_bits(par, n)
        q = self.rope(q.reshape(T, nq * d), pos, nq).reshape(T, nq, d)
        k = self.rope(k.reshape(T, nkv * d), pos, nkv).reshape(T, nkv, d)
        for r in range(b):
            for i in range(n):
                kc[r, :, prefix[r] + i] = k[r * n + i]
                vc[r, :, prefix[r] + i] = v[r * n + i]
        attn = self.attention(q, kc, vc, mbits, prefix, n)
        x = x + self.gemm(attn.reshape(T, nq * d), self.wo(l))
        xn2 = self.rmsnorm(x)
        lg = self.router_logits(xn2, l)
        ids, w = self.topk(lg)
        off, perm, pos_p = self.permute(ids)
        sh = self.shared(l)
        if sh is not None:  # x += shared SwiGLU (fp32), before the routed sum
            Ysh = np.zeros((T, s.hidden), np.float32)
            O.lib().orc_expert_swiglu(O._ptr(np.ascontiguousarray(xn2)), T, s.hidden, s.shared_inter, O._ptr(sh[0]),
                                      O._ptr(sh[1]), O._ptr(sh[2]), O._ptr(Ysh))
            x = (x + Ysh).astype(np.float32)
        y = self.moe(xn2, l, ids, w)
        x_out = (x.astype(np.float64) + y).astype(np.float32)
        return x_out, dict(xn1=xn1, q=q, attn=attn, xn2=xn2, logits_r=lg, ids=ids, weights=w, offsets=off,
                           pos=pos_p, x_mid=x)

    def head(self, x):
        xf = self.rmsnorm(x)
        logits = self.gemm(xf, self.lm_head())
        return xf, logits


# ------------------------------------------------------------------ drafter
# (engine.cu tid::draft: layer l base 700000 + 100 l; +1 Wqkv, +2 Wo, +3 W1,
# +4 W3, +5 W2 — dense decoder layers sharing the target's embed / LM head)
def _draft_tid(l):
    return 700000 + 100 * l


def draft_weights(om, l):
    s = om.s
    key = ("draft", l)
    if key not in om._cache:
        h, di, k = s.hidden, s.draft_inter, s.n_q_heads * s.head_dim
        b = _draft_tid(l)
        om._cache[key] = (om._fill(om.qkv_w * h, b + 1, math.sqrt(3.0 / h)).reshape(om.qkv_w, h),
                          om._fill(h * k, b + 2, math.sqrt(3.0 / k)).reshape(h, k),
                          om._fill(di * h, b + 3, math.sqrt(3.0 / h)).reshape(di, h),
                          om._fill(di * h, b + 4, math.sqrt(3.0 / h)).reshape(di, h),
                          om._fill(h * di, b + 5, math.sqrt(3.0 / di)).reshape(h, di))
    return om._cache[key]


def attn_block(om, x, wqkv, wo, kc, vc, prefix, n):
    """x + Wo·attn(RoPE(Wqkv·rmsnorm(x))) for a batch of chains (rows r*n+i
    at prefix[r]+i); K/V appended to kc/vc [b, n_kv, s_max, d] in place."""
    s = om.s
    b = len(prefix)
    T = b * n
    d, nq, nkv = s.head_dim, s.n_q_heads, s.n_kv_heads
    qkv = O.f32_to_bf16(om.gemm(om.rmsnorm(x), wqkv)).reshape(T, -1)
    pos = np.concatenate([prefix[r] + np.arange(n) for r in range(b)]).astype(np.int32)
    q = om.rope(qkv[:, :nq * d], pos, nq).reshape(T, nq, d)
    k = om.rope(qkv[:, nq * d:(nq + nkv) * d], pos, nkv).reshape(T, nkv, d)
    v = qkv[:, (nq + nkv) * d:].reshape(T, nkv, d)
    for r in range(b):
        for i in range(n):
            kc[r, :, prefix[r] + i] = k[r * n + i]
            vc[r, :, prefix[r] + i] = v[r * n + i]
    mbits = np.tile(om.mask_bits(None, n), b)
    attn = om.attention(q, kc, vc, mbits, np.asarray(prefix, np.int32), n)
    return (x + om.gemm(attn.reshape(T, nq * d), wo)).astype(np.float32)


def swiglu_dense(om, x, w1, w3, w2):
    """x + W2·bf16(silu(W1·xn)·(W3·xn)) with xn = rmsnorm(x) (fp32 out)."""
    xn = om.rmsnorm(x)
    y = np.zeros((x.shape[0], om.s.hidden), np.float32)
    O.lib().orc_expert_swiglu(O._ptr(np.ascontiguousarray(xn)), x.shape[0], om.s.hidden, w1.shape[0], O._ptr(w1),
                              O._ptr(w3), O._ptr(w2), O._ptr(y))
    return (x + y).astype(np.float32)


class OracleDecoder:
    """Greedy autoregressive decoding of ONE request by the CPU oracle: the
    sequence every speculative decode must commit under greedy verification
    (acceptance only decides how many of these tokens one step commits)."""

    def __init__(self, om, s_max):
        s = om.s
        self.om, self.s_max = om, s_max
        shape = (1, s.n_kv_heads, s_max, s.head_dim)
        self.kc = [np.zeros(shape, np.uint16) for _ in range(s.n_layers)]
        self.vc = [np.zeros(shape, np.uint16) for _ in range(s.n_layers)]
        self.len = 0

    def run(self, tokens):
        """Feed tokens (a chain) at the current position; returns fp32 logits [n, V]."""
        om = self.om
        n = len(tokens)
        x = O.bf16_to_f32(om.embed()[np.asarray(tokens)]).astype(np.float32)
        for l in range(om.s.n_layers):
            x, _ = om.layer(l, x, self.kc[l], self.vc[l], np.array([self.len], np.int32), n)
        self.len += n
        return om.head(x)[1]

    def prefill(self, prompt, chunk):
        logits = None
        for c in range(0, len(prompt), chunk):
            logits = self.run(prompt[c:c + chunk])
        return logits[-1]

    @staticmethod
    def margin(logits_row):
        top = np.sort(logits_row)[-2:]
        return float(top[1] - top[0]) / float(np.std(logits_row) + 1e-30)

    def greedy(self, prompt, steps, chunk):
        """(tokens: the greedy next token after the prompt then `steps` more,
        margins: top-1 minus top-2 logit over the logit std for each)."""
        lg = self.prefill(list(prompt), chunk)
        toks, margins = [int(np.argmax(lg))], [self.margin(lg)]
        for _ in range(steps):
            lg = self.run([toks[-1]])[-1]
            toks.append(int(np.argmax(lg)))
            margins.append(self.margin(lg))
        return toks, margins
