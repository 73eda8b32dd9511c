import os, sys, numpy as np
sys.path.insert(0, os.getcwd())
from paper_2508_21706_b200.engine import VerifyEngine, TINY
import dataclasses
s = dataclasses.replace(TINY, seed=0x5EED + 3, lm_scale=8.0, router_scale=4.0)
for pf in ("0", "1"):
    os.environ["SMO_B1_PREFETCH"] = pf
    eng = VerifyEngine(s, max_batch=1, max_verify=2, max_seq=512, batch_one=True, compress_experts=True)
    prefix = np.array([300], np.int32)
    eng.fill_prefix(prefix)
    rows = []
    for i in range(5):
        eng.verify(np.array([[17 + i, 4242 - i]], np.int32), prefix)
        t = eng.last_times()
        rows.append((round(t["h2d_bytes"] / 1e6, 3), round(t["target_total"] * 1e3, 3)))
    print(pf, rows)
    eng.close()
