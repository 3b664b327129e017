"""Time fused add, compress and decompress of several library builds
(VC3_B200_LIB) on 2^28 vectors: grid-cap sweeps."""
import os
import subprocess
import sys

CODE = r'''
import sys, torch
sys.path.insert(0, ".")
import paper_2003_02633_b200 as vc3b
from paper_2003_02633_b200 import _native
lib = _native.load(); dev = torch.device("cuda", 0)
n = 1 << 28
g = torch.Generator(device=dev).manual_seed(1)
va = torch.rand((n, 3), device=dev, generator=g) * 2 - 1
a = vc3b.compress(va, vc3b.DEFAULT_LAYOUT, vc3b.ALL_SINGLE_POLICY)
b = vc3b.compress(torch.rand((n, 3), device=dev, generator=g) * 2 - 1, vc3b.DEFAULT_LAYOUT, vc3b.ALL_SINGLE_POLICY)
c = torch.empty_like(a); vo = torch.empty_like(va)
cl = _native.c_layout(vc3b.DEFAULT_LAYOUT); s = torch.cuda.current_stream().cuda_stream
fa = lambda: lib.vc3_add_compressed(a.data_ptr(), b.data_ptr(), c.data_ptr(), n, cl, 7, s)
fc = lambda: lib.vc3_compress(va.data_ptr(), c.data_ptr(), n, cl, 7, None, s)
fd = lambda: lib.vc3_decompress(a.data_ptr(), vo.data_ptr(), n, cl, s)
res = []
for name, f in (("add", fa), ("compress", fc), ("decompress", fd)):
    for _ in range(5): f()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); [f() for _ in range(30)]; e1.record(); e1.synchronize()
    ms = e0.elapsed_time(e1) / 30
    res.append(f"{name} {n / ms / 1e6:.1f}")
print(sys.argv[1], "  ".join(res), "Gvec/s")
'''

for lib in sys.argv[1:]:
    env = dict(os.environ, VC3_B200_LIB=os.path.abspath(lib), VC3_B200_AUTOBUILD="0")
    subprocess.run([sys.executable, "-c", CODE, lib], env=env, check=False)
