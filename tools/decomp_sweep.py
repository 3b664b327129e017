"""Time decompress of several library builds (VC3_B200_LIB) on 2^28 words."""
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
a = vc3b.compress(torch.rand((n, 3), device=dev, generator=g) * 2 - 1, vc3b.DEFAULT_LAYOUT, vc3b.ALL_SINGLE_POLICY)
out = torch.empty((n, 3), device=dev)
cl = _native.c_layout(vc3b.DEFAULT_LAYOUT); s = torch.cuda.current_stream().cuda_stream
f = lambda: lib.vc3_decompress(a.data_ptr(), out.data_ptr(), n, cl, s)
for _ in range(5): f()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); [f() for _ in range(30)]; e1.record(); e1.synchronize()
ms = e0.elapsed_time(e1) / 30
ref = vc3b.decompress(a[:4096].cpu().numpy())
assert (out[:4096].cpu().numpy() == ref).all()
print(f"{sys.argv[1]}: {ms:.3f} ms  {n / ms / 1e6:.1f} Gword/s  {20 * n / ms / 1e6:.0f} GB/s")
'''

for lib in sys.argv[1:]:
    env = dict(os.environ, VC3_B200_LIB=os.path.abspath(lib), VC3_B200_AUTOBUILD="0")
    subprocess.run([sys.executable, "-c", CODE, lib], env=env, check=False)
