import sys, os
sys.path.insert(0, os.path.join(os.environ.get("GRAFT_REPO_ROOT", "."), "tools"))
import kbench
b, n, s = (int(v) for v in sys.argv[1:4])
print(kbench.attn(b, n, s))
