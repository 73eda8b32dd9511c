"""Generate tests/golden/reference_vectors.json from the UNMODIFIED reference.

Run here (where /root/reference exists): `python oracle/gen_golden.py`.
Inputs come from the restated `verify-attention --random` generator
(moeplan.cpp:287-311, oracle.c:orc_random_cases), which is itself pinned by the
survey's Appendix B values recorded below; outputs come from the reference's
own moeplan::chunked_attention / simulate_tokens / splitmix64 via
oracle/_ref/libmoeplan_ref.so. The committed JSON lets the oracle and the GPU
parity tests run where /root/reference is absent (the GPU box).
"""
import ctypes as C
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import oracle_py as O  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                   "reference_vectors.json")


def ref_attention(c):
    R = O.ref()
    out = np.zeros((c["n"], c["d"]))
    Q, K, V = (np.ascontiguousarray(c[x]) for x in "QKV")
    m = np.ascontiguousarray(c["mask"], np.uint8)
    rc = R.ref_chunked_attention(c["n"], c["p"], c["d"], O._ptr(Q), O._ptr(K), O._ptr(V), c["n"], O._ptr(m), O._ptr(out))
    assert rc == 0, R.ref_last_error()
    return out


def main():
    O.build()
    R = O.ref()
    g = {"source": "reference headers /root/reference/proj/include via oracle/ref_shim.cpp",
         "splitmix64": {str(x): R.ref_splitmix64(x) for x in (0, 1, 42, 7, 2**64 - 1)}}
    stream = np.zeros(8)
    R.ref_trial_stream(R.ref_splitmix64(42), 8, O._ptr(stream))
    g["trial_stream_splitmix42"] = stream.tolist()
    cases = {}
    for seed, count in ((42, 50), (7, 50), (2024, 20)):
        cs = O.random_cases(seed, count)
        outs = [ref_attention(c) for c in cs]
        cases[str(seed)] = {
            "count": count,
            "dims": [[c["n"], c["p"], c["d"]] for c in cs],
            "Q00": [float(c["Q"][0, 0]) for c in cs],
            "mask_rows": [c["mask"].astype(int).tolist() for c in cs],
            "out": [o.tolist() for o in outs],
            "sum": float(sum(o.sum() for o in outs)),
            "rows": int(sum(o.shape[0] for o in outs)),
        }
    g["random_cases"] = cases
    sims = []
    for p in (0.5, 0.8):
        for k in (1, 4, 10):
            mean, sd = C.c_double(), C.c_double()
            probs = np.full(10, p)
            R.ref_simulate_tokens(O._ptr(probs), 10, k, 100000, k * 1000 + 7, C.byref(mean), C.byref(sd))
            sims.append({"p": p, "k": k, "trials": 100000, "seed": k * 1000 + 7,
                         "mean": mean.value, "std": sd.value})
    g["simulate_tokens"] = sims
    g["mask_memory_savings"] = {"5,1590": R.ref_mask_memory_savings(5, 1590),
                                "5,0": R.ref_mask_memory_savings(5, 0)}
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    with open(OUT, "w") as f:
        json.dump(g, f)
    print("wrote", OUT, os.path.getsize(OUT), "bytes")
    c42 = cases["42"]
    print("seed42 sum", repr(c42["sum"]), "rows", c42["rows"], "case0", c42["dims"][0], c42["Q00"][0], c42["out"][0][0][0])
    print("seed7 sum", repr(cases["7"]["sum"]), "rows", cases["7"]["rows"])


if __name__ == "__main__":
    main()
