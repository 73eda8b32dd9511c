#!/bin/bash
# K1 same-box A/B: tools/k1_ab.sh <lib.so>... — kbench attn at a few shapes per library (default lib first)
for lib in default "$@"; do
  if [ "$lib" = default ]; then unset SPECMOE_LIB; else export SPECMOE_LIB=$lib; fi
  echo "== $lib"
  timeout 120 python - <<'PY'
import sys, os, json
sys.path.insert(0, "tools")
import kbench
for b, n, s in ((1, 9, 1024), (16, 9, 1024), (32, 9, 1024), (64, 16, 1024), (32, 9, 4096)):
    r = kbench.attn(b, n, s)
    print(json.dumps({k: (round(v, 3) if isinstance(v, float) else v) for k, v in r.items() if k in ("b", "n", "s", "us", "frac")}))
PY
done
