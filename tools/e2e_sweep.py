"""Time the host-buffer fused add (vc3_add_compressed_host, pinned buffers,
2^28 vectors) of several library builds (VC3_B200_LIB)."""
import os
import subprocess
import sys

CODE = r'''
import sys, time, torch, numpy as np
sys.path.insert(0, ".")
import paper_2003_02633_b200 as vc3b
from paper_2003_02633_b200 import _native
lib = _native.load()
n = 1 << 28
ha = torch.randint(0, 2**62, (n,), dtype=torch.int64).pin_memory()
hb = torch.randint(0, 2**62, (n,), dtype=torch.int64).pin_memory()
hc = torch.empty(n, dtype=torch.int64).pin_memory()
cl = _native.c_layout(vc3b.DEFAULT_LAYOUT)
f = lambda: lib.vc3_add_compressed_host(ha.data_ptr(), hb.data_ptr(), hc.data_ptr(), n, cl, 7, 0)
f()
t0 = time.perf_counter()
for _ in range(5): f()
dt = (time.perf_counter() - t0) / 5
print(f"{sys.argv[1]}: {dt*1e3:.1f} ms  {n/dt/1e9:.2f} Gvec/s  H2D {16*n/dt/1e9:.1f} GB/s")
'''

for lib in sys.argv[1:]:
    env = dict(os.environ, VC3_B200_LIB=os.path.abspath(lib), VC3_B200_AUTOBUILD="0")
    subprocess.run([sys.executable, "-c", CODE, lib], env=env, check=False)
