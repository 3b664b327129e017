"""Small workload touching every kernel family once, for compute-sanitizer
(memcheck / racecheck / synccheck, one tool per run):

    compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_run.py

K1 compress (fast all-single and generic policies, wide layout), K2
decompress (exact / contract, table and wide layouts), K3 fused add, K4 axpy
and RK stage (fast path and a generic policy, both modes), K5 fp32
baselines, K6 error statistics, K7 variants, the host-buffer pipeline
(pinned and pageable), FR divergence (tcgen05 dense and sum-factorised).
Sizes are a few thousand vectors (ragged, so every tail loop runs).
"""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import paper_2003_02633_b200 as vc3b  # noqa: E402
from paper_2003_02633_b200 import fr, ops, variants  # noqa: E402
from paper_2003_02633_b200.layout import BitLayout, PrecisionPolicy  # noqa: E402

dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(11)
n = 4099
lays = [vc3b.DEFAULT_LAYOUT, BitLayout(0, 7, 22, 10, 25, 80)]
pols = [vc3b.ALL_SINGLE_POLICY, PrecisionPolicy("single", "double", "single")]
v = torch.rand((n, 3), device=dev, generator=g) * 2 - 1
v[::17] = 0.0
v[5::31, 2] = -0.0
for lay in lays:
    for pol in pols:
        a = vc3b.compress(v, lay, pol)
        b = vc3b.compress(v.flip(0).contiguous(), lay, pol)
        for mode in ("exact", "contract"):
            vc3b.decompress(a, lay, mode=mode)
            ops.add_compressed(a, b, lay, pol, mode=mode)
            ops.axpy(0.5, a, b, lay, pol, mode=mode)
            q, dq = a.clone(), b.clone()
            ops.rk_stage(0.5, 0.25, 1e-3, q, dq, a, lay, pol, mode=mode)
        vc3b.compress(v[1:], lay, pol)  # misaligned: scalar paths
        ops.add_compressed(a[1:], b[1:], lay, pol)
ops.add_raw(v, v)
w = vc3b.compress(v, vc3b.DEFAULT_LAYOUT, vc3b.ALL_SINGLE_POLICY)
vc3b.magnitude_event_counts(v)
# host-buffer pipeline: pageable and pinned
hv = v.cpu().numpy()
hw = vc3b.compress(hv, vc3b.DEFAULT_LAYOUT, vc3b.ALL_SINGLE_POLICY)
vc3b.decompress(hw)
ops.add_compressed(hw, hw[::-1].copy())
pa = torch.from_numpy(hw.view(np.int64)).pin_memory().numpy().view(np.uint64)
ops.add_compressed(pa, pa)
# K6 error statistics and K7 variants
from paper_2003_02633_b200 import analysis  # noqa: E402

vh = vc3b.decompress(w)
lib = vc3b._native.load()
for kind in range(4):
    out = torch.empty(4, dtype=torch.float64, device=dev)
    lib.vc3_error_stats(v.data_ptr(), vh.data_ptr(), n, kind, 1 << 20, out.data_ptr(),
                        torch.cuda.current_stream().cuda_stream)
for var in (variants.Compander("uniform"), variants.Compander("cosine"), variants.Compander("tanh", 2.0),
            variants.SplitConfig(35, 98303)):
    ww = variants.compress_variant(v, var)
    variants.decompress_variant(ww, var)
# FR divergence: dense tcgen05 (k = 4) and sum-factorised (k = 1..4)
for k, ne in ((4, 300), (1, 37)):
    ns = (k + 1) ** 3
    rng = np.random.default_rng(k)
    F = torch.from_numpy(rng.uniform(-1, 1, (ns, 2, ne, 3)).astype(np.float32)).to(dev)
    words = vc3b.compress(F.reshape(-1, 3), vc3b.DEFAULT_LAYOUT, vc3b.ALL_SINGLE_POLICY).reshape(ns, 2, ne)
    op = fr.Operator(fr.divergence_operator(k))
    fr.flux_divergence(words, op)
    fr.flux_divergence_f32(F, op)
    fr.flux_divergence_hex(words)
    fr.flux_divergence_hex_f32(F)
torch.cuda.synchronize()
print("sanitize workload ok")
