"""Time the K7 variant kernels (compress / decompress) on 2^28 cube vectors."""
import sys
sys.path.insert(0, ".")
import torch
import paper_2003_02633_b200 as vc3b
from paper_2003_02633_b200 import variants

n = 1 << 28
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(3)
v = torch.rand((n, 3), device=dev, generator=g) * 2 - 1


def t(fn, it=5):
    fn(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(it):
        fn()
    e.record(); e.synchronize()
    return s.elapsed_time(e) / it * 1e-3


for var in (variants.Compander("uniform"), variants.Compander("cosine"), variants.Compander("tanh", 2.0),
            variants.SplitConfig(35, 98303)):
    w = variants.compress_variant(v, var)
    tc = t(lambda: variants.compress_variant(v, var))
    td = t(lambda: variants.decompress_variant(w, var))
    print(f"{var}: compress {n / tc / 1e9:.1f} Gvec/s, decompress {n / td / 1e9:.1f} Gvec/s")
