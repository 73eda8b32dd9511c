python - <<'PY'
import sys, json
sys.argv=['kbench','attn']
sys.path.insert(0,'tools')
import kbench as K
for (b,n,s) in [(1,5,1024),(1,9,1024),(4,9,1024),(32,9,1024),(32,5,1024),(64,9,4096),(16,9,16384)]:
    r=K.attn(b,n,s); print(json.dumps({k:(round(v,3) if isinstance(v,float) else v) for k,v in r.items()}))
PY
