"""Cost of cudaHostRegister / Unregister on pageable numpy memory (probe for
the pageable host-buffer path)."""
import ctypes, time
import numpy as np
import torch

torch.cuda.init()
cr = ctypes.CDLL("libcudart.so.12") if False else None
rt = torch.cuda.cudart()
n = 1 << 28
a = np.ones(n, dtype=np.uint64)  # 2 GiB, touched
for chunk_log2 in (21, 24, 28):
    cb = (1 << chunk_log2) * 8
    t0 = time.perf_counter()
    m = 0
    for off in range(0, n * 8, cb):
        p = a.ctypes.data + off
        rt.cudaHostRegister(p, cb, 0)
        rt.cudaHostUnregister(p)
        m += cb
        if m >= (1 << 31):
            break
    dt = time.perf_counter() - t0
    print(f"register+unregister chunks of {cb >> 20} MiB: {m / dt / 1e9:.1f} GB/s")
t0 = time.perf_counter(); b = a.copy(); dt = time.perf_counter() - t0
print(f"numpy copy 1 thread: {a.nbytes / dt / 1e9:.1f} GB/s")
