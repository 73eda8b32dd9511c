for q in 0 9 12 14 16 18 27; do
  if [ $q = 0 ]; then unset SMO_ATTN_Q; else export SMO_ATTN_Q=$q; fi
  python - <<'PY'
import os, sys, json
sys.path.insert(0, "tools"); sys.argv = ["kbench"]
import kbench as K
for (b, n, s) in ((32, 9, 1024), (32, 5, 1024), (64, 1, 4096), (16, 8, 4096)):
    r = K.attn(b, n, s)
    print(os.environ.get("SMO_ATTN_Q", "auto"), json.dumps(r))
PY
done
timeout 900 python tools/probe_box.py > /dev/null 2>&1; cat gpurun_out/probe_box.json | head -c 3000
