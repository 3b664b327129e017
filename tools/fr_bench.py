"""Time the FR flux-divergence kernels (compressed vs float32) on one GPU."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2003_02633_b200 import codec, fr  # noqa: E402


def timeit(fn, iters=20):
    fn(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record(); e.synchronize()
    return s.elapsed_time(e) / iters * 1e-3


def main(k=4, n_elem=1 << 18, n_vars=5):
    ns = (k + 1) ** 3
    D = fr.divergence_operator(k)
    op = fr.Operator(D)
    g = torch.Generator(device="cuda").manual_seed(0)
    F = torch.rand((ns, n_vars, n_elem, 3), device="cuda", generator=g) * 2 - 1
    words = codec.compress(F.reshape(-1, 3)).reshape(ns, n_vars, n_elem)
    rows = n_elem * n_vars
    t_c = timeit(lambda: fr.flux_divergence(words, op))
    t_f = timeit(lambda: fr.flux_divergence_f32(F, op))
    if k <= 4:
        t_hc = timeit(lambda: fr.flux_divergence_hex(words))
        t_hf = timeit(lambda: fr.flux_divergence_hex_f32(F))
        for name, t, b in (("hex-comp", t_hc, ns * 12), ("hex-f32", t_hf, ns * 16)):
            print(f"{name:10s} k={k} n_elem={n_elem} {t*1e3:8.3f} ms  {rows/t/1e9:7.3f} G elem-eq/s  "
                  f"{b*rows/t/1e9:7.1f} GB/s")
    flops = 2.0 * 3 * ns * ns * rows
    for name, t, b in (("compressed", t_c, 8 * 3 * 0 + ns * 8 + ns * 4), ("f32", t_f, ns * 12 + ns * 4)):
        print(f"{name:10s} k={k} n_elem={n_elem} {t*1e3:8.3f} ms  {rows/t/1e9:7.3f} G elem-eq/s  "
              f"{flops/t/1e12:7.1f} TFLOP/s (x3 on tensor)  {b*rows/t/1e9:7.1f} GB/s")


if __name__ == "__main__":
    for k, n in ((4, 1 << 18), (3, 1 << 19), (5, 1 << 17), (2, 1 << 20), (1, 1 << 21)):
        main(k, n)
