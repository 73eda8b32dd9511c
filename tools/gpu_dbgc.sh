timeout 300 python tools/dbg_cpuattn2.py 2>&1 | tail -14
