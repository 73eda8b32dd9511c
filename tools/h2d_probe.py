"""Host->device link probe: pinned H2D GB/s for one vs several concurrent
copy streams, portable vs write-combined pinned memory (cudart via ctypes so
the allocation flags are explicit). Prints JSON lines."""
import ctypes as C
import json

import torch

cudart = C.CDLL("libcudart.so.12") if False else None
try:
    cudart = C.CDLL("libcudart.so")
except OSError:
    import glob
    cands = glob.glob("/usr/local/cuda/lib64/libcudart.so*")
    cudart = C.CDLL(cands[0])

SIZE = 1 << 31  # 2 GiB
dev = torch.device("cuda:0")
dst = torch.empty(SIZE, dtype=torch.uint8, device=dev)
for flags, name in ((1, "portable"), (1 | 4, "portable+writecombined")):
    hp = C.c_void_p()
    assert cudart.cudaHostAlloc(C.byref(hp), C.c_size_t(SIZE), C.c_uint(flags)) == 0
    C.memset(hp, 1, SIZE)
    for nstreams in (1, 2, 4):
        streams = [torch.cuda.Stream() for _ in range(nstreams)]
        chunk = SIZE // nstreams
        best = 0.0
        for rep in range(4):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for i, st in enumerate(streams):
                st.wait_event(e0)
                cudart.cudaMemcpyAsync(C.c_void_p(dst.data_ptr() + i * chunk), C.c_void_p(hp.value + i * chunk),
                                       C.c_size_t(chunk), 1, C.c_void_p(st.cuda_stream))
            for st in streams:
                ev = torch.cuda.Event()
                ev.record(st)
                torch.cuda.current_stream().wait_event(ev)
            e1.record()
            torch.cuda.synchronize()
            gbs = SIZE / (e0.elapsed_time(e1) * 1e-3) / 1e9
            best = max(best, gbs) if rep else best
        print(json.dumps({"memory": name, "streams": nstreams, "h2d_gbs": round(best, 2)}), flush=True)
    cudart.cudaFreeHost(hp)
