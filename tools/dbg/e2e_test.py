import sys, time, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_2003_02633_b200 as vc3b
from paper_2003_02633_b200 import _native
lib = _native.load(); lay, pol = vc3b.DEFAULT_LAYOUT, vc3b.ALL_SINGLE_POLICY; cl = _native.c_layout(lay)
n = 1 << 28
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(1)
a = vc3b.compress(torch.rand((n, 3), device=dev, generator=g) * 2 - 1, lay, pol)
b = vc3b.compress(torch.rand((n, 3), device=dev, generator=g) * 2 - 1, lay, pol)
c = vc3b.add_compressed(a, b, lay, pol)
pin = [torch.empty(n, dtype=torch.uint64, pin_memory=True) for _ in range(3)]
pin[0].copy_(a); pin[1].copy_(b)
pg = [np.empty(n, dtype=np.uint64) for _ in range(3)]
pg[0][:] = pin[0].numpy(); pg[1][:] = pin[1].numpy()
for name, bufs in (("pinned", [t.numpy() for t in pin]), ("pageable", pg)):
    f = lambda: lib.vc3_add_compressed_host(bufs[0].ctypes.data, bufs[1].ctypes.data, bufs[2].ctypes.data, n, cl, pol.mask, 0)
    f(); t0 = time.perf_counter()
    for _ in range(3): f()
    dt = (time.perf_counter() - t0) / 3
    print(name, n / dt / 1e9, "Gvec/s", np.array_equal(bufs[2], c.cpu().numpy()))
# compress / decompress host pageable
v = (torch.rand((n // 4, 3), device=dev, generator=g) * 2 - 1).cpu().numpy()
t0 = time.perf_counter(); w = vc3b.compress(v, lay, pol); dt = time.perf_counter() - t0
print("compress host pageable", v.shape[0] / dt / 1e9, np.array_equal(w, vc3b.compress(torch.from_numpy(v).to(dev), lay, pol).cpu().numpy()))
t0 = time.perf_counter(); vv = vc3b.decompress(w, lay); dt = time.perf_counter() - t0
print("decompress host pageable", v.shape[0] / dt / 1e9, np.array_equal(vv, vc3b.decompress(torch.from_numpy(w).to(dev), lay).cpu().numpy()))
