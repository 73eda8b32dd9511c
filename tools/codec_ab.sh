#!/bin/bash
# Unary decoder same-box A/B: tools/codec_ab.sh <lib.so>... — one Mixtral block, uniform and gaussian-like,
# libraries alternated three times (default library = "default")
for rep in 1 2 3; do
  for lib in default "$@"; do
    if [ "$lib" = default ]; then unset SPECMOE_LIB; else export SPECMOE_LIB=$lib; fi
    timeout 120 python - "$lib" <<'PY'
import sys, json
sys.path.insert(0, "tools")
import kbench
u = kbench.codec(bits=1); g = kbench.codec(bits=1, dist="gaussian")
print(json.dumps({"lib": sys.argv[1], "uniform_us": round(u["us"], 1), "uniform_frac": round(u["frac"], 3),
                  "gauss_us": round(g["us"], 1)}))
PY
  done
done
