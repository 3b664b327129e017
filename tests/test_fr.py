"""FR flux divergence (Alg. 1).

CPU: the operator construction (exact on polynomials of degree <= k).
GPU: the tcgen05 kernel against a float64 contraction of the decompressed
fluxes (the oracle decodes the words bit-exactly), on the compressed and
the float32 paths, ragged element counts, padded strides, ns = 8 .. 216.
Tolerance: 3xTF32 products accumulate in fp32, so each output is checked
to 2^-18 of sum_j,d |D| |X| (the fp32 sum itself carries ~ns * 2^-24)."""

from pathlib import Path

import numpy as np
import pytest

from conftest import layout_by_name, policy_by_code
from paper_2003_02633_b200 import fr


@pytest.mark.parametrize("k", [1, 2, 4, 5])
def test_operator_exact_on_polynomials(k):
    D = fr.divergence_operator(k, dtype=np.float64)
    ns = (k + 1) ** 3
    x, y, z = fr.solution_points(k).T
    F = np.stack([x ** k * y, y ** (k - 1) * z + x, z ** k - y ** 2], axis=1)  # degree <= k per direction
    div = np.einsum("djk,jd->k", D.reshape(3, ns, ns), F)
    want = k * x ** (k - 1) * y + (k - 1) * y ** max(k - 2, 0) * z * (k > 1) + k * z ** (k - 1)
    np.testing.assert_allclose(div, want, atol=1e-9 * ns)


def _reference(D, X):
    """float64 div[k][c][i] and the error scale sum |D||X|."""
    ns = D.shape[1]
    D3 = D.astype(np.float64).reshape(3, ns, ns)  # [d][j][k]
    X = X.astype(np.float64)                      # [j][c][i][d]
    ref = np.einsum("djk,jcid->kci", D3, X)
    scale = np.einsum("djk,jcid->kci", np.abs(D3), np.abs(X))
    return ref, scale


def _check(got, ref, scale, what):
    err = np.abs(got.astype(np.float64) - ref)
    bound = 2.0 ** -18 * scale + 1e-30
    worst = float((err / bound).max())
    assert worst <= 1.0, f"{what}: worst error {worst:.3f} x bound"


@pytest.mark.gpu
@pytest.mark.parametrize("k,n_elem,n_vars,pad", [(4, 1000, 5, 0), (4, 128, 1, 0), (1, 37, 2, 3),
                                                  (2, 300, 3, 17), (5, 260, 2, 0), (4, 1, 5, 0)])
def test_fr_divergence_matches_float64(oracle, vc3b, cuda, k, n_elem, n_vars, pad):
    import torch

    rng = np.random.default_rng(100 + k + n_elem)
    ns = (k + 1) ** 3
    ld = n_elem + pad
    D = rng.standard_normal((3 * ns, ns)).astype(np.float32)
    F = rng.uniform(-2, 2, (ns, n_vars, ld, 3)).astype(np.float32)
    F[:, :, ::7] *= 1e-3          # mixed magnitudes
    F[:, :, 5::11] = 0.0          # zero vectors
    lay = vc3b.DEFAULT_LAYOUT
    words = oracle.compress(F.reshape(-1, 3), lay, policy_by_code("SSS")).reshape(ns, n_vars, ld)
    X = oracle.decompress(words.reshape(-1), lay).reshape(ns, n_vars, ld, 3)
    op = fr.Operator(D)
    got = fr.flux_divergence(torch.from_numpy(words.view(np.int64)).cuda().view(torch.uint64), op,
                             n_elem).cpu().numpy()
    ref, scale = _reference(D, X[:, :, :n_elem])
    _check(got[:, :, :n_elem], ref, scale, f"compressed k={k}")
    got32 = fr.flux_divergence_f32(torch.from_numpy(F).cuda(), op, n_elem).cpu().numpy()
    ref32, scale32 = _reference(D, F[:, :, :n_elem])
    _check(got32[:, :, :n_elem], ref32, scale32, f"f32 k={k}")


@pytest.mark.gpu
def test_fr_divergence_physical_operator_and_layouts(oracle, vc3b, cuda):
    """The degree-4 hexahedron operator on a smooth field, two layouts
    (table and wide-angle decode paths)."""
    import torch

    k, n_elem, n_vars = 4, 2000, 5
    ns = 125
    D = fr.divergence_operator(k)
    xyz = fr.solution_points(k)
    rng = np.random.default_rng(9)
    a = rng.uniform(0.5, 1.5, (n_vars, n_elem))
    F = np.empty((ns, n_vars, n_elem, 3), np.float32)
    F[..., 0] = np.sin(xyz[:, 0])[:, None, None] * a
    F[..., 1] = (xyz[:, 1] ** 2)[:, None, None] * a
    F[..., 2] = np.cos(xyz[:, 2])[:, None, None] + 0 * a
    op = fr.Operator(D)
    for lname in ("17_18", "wide_10_25"):
        lay = layout_by_name(lname)
        words = oracle.compress(F.reshape(-1, 3), lay, policy_by_code("SSS")).reshape(ns, n_vars, n_elem)
        X = oracle.decompress(words.reshape(-1), lay).reshape(ns, n_vars, n_elem, 3)
        got = fr.flux_divergence(torch.from_numpy(words.view(np.int64)).cuda().view(torch.uint64),
                                 op, layout=lay).cpu().numpy()
        ref, scale = _reference(D, X)
        _check(got, ref, scale, lname)


@pytest.mark.gpu
@pytest.mark.parametrize("k,n_elem,n_vars,pad", [(4, 1000, 5, 0), (1, 37, 2, 3), (2, 300, 3, 17),
                                                  (3, 129, 1, 0)])
def test_fr_divergence_hex_matches_dense(oracle, vc3b, cuda, k, n_elem, n_vars, pad):
    """The sum-factorised hexahedron kernel == Alg. 1 with the dense operator."""
    import torch

    rng = np.random.default_rng(200 + k)
    ns, ld = (k + 1) ** 3, n_elem + pad
    F = rng.uniform(-2, 2, (ns, n_vars, ld, 3)).astype(np.float32)
    F[:, :, 3::13] = 0.0
    lay = vc3b.DEFAULT_LAYOUT
    words = oracle.compress(F.reshape(-1, 3), lay, policy_by_code("SSS")).reshape(ns, n_vars, ld)
    X = oracle.decompress(words.reshape(-1), lay).reshape(ns, n_vars, ld, 3)
    D = fr.divergence_operator(k, dtype=np.float64)
    # the kernel takes the float32 1D matrix: compare against the operator it implies
    m32 = fr.lagrange_derivative_matrix(fr.gauss_legendre_nodes(k)).astype(np.float32)
    D32 = fr.divergence_operator(k, dtype=np.float64)
    n = k + 1
    eye = np.eye(n)
    M = m32.astype(np.float64)
    D32 = np.concatenate([np.kron(eye, np.kron(eye, M)).T, np.kron(eye, np.kron(M, eye)).T,
                          np.kron(M, np.kron(eye, eye)).T], axis=0)
    assert np.abs(D32 - D).max() < 1e-5
    got = fr.flux_divergence_hex(torch.from_numpy(words.view(np.int64)).cuda().view(torch.uint64),
                                 n_elem).cpu().numpy()
    ref, scale = _reference(D32, X[:, :, :n_elem])
    _check(got[:, :, :n_elem], ref, scale, f"hex k={k}")
    got32 = fr.flux_divergence_hex_f32(torch.from_numpy(F).cuda(), n_elem).cpu().numpy()
    ref32, scale32 = _reference(D32, F[:, :, :n_elem])
    _check(got32[:, :, :n_elem], ref32, scale32, f"hex f32 k={k}")


@pytest.mark.gpu
@pytest.mark.parametrize("ns,n_elem,n_vars", [(1, 300, 2), (37, 513, 3), (256, 260, 1), (125, 0, 5)])
def test_fr_divergence_generic_operator_shapes(oracle, vc3b, cuda, ns, n_elem, n_vars):
    """Alg. 1 with any dense operator: non-cube point counts, the 256-point
    maximum, an empty element range."""
    import torch

    rng = np.random.default_rng(ns + n_elem)
    D = rng.standard_normal((3 * ns, ns)).astype(np.float32)
    ld = max(n_elem, 1)
    F = rng.uniform(-1, 1, (ns, n_vars, ld, 3)).astype(np.float32)
    lay = vc3b.DEFAULT_LAYOUT
    words = oracle.compress(F.reshape(-1, 3), lay, policy_by_code("SSS")).reshape(ns, n_vars, ld)
    X = oracle.decompress(words.reshape(-1), lay).reshape(ns, n_vars, ld, 3)
    op = fr.Operator(D)
    got = fr.flux_divergence(torch.from_numpy(words.view(np.int64)).cuda().view(torch.uint64), op,
                             n_elem).cpu().numpy()
    if n_elem:
        ref, scale = _reference(D, X[:, :, :n_elem])
        _check(got[:, :, :n_elem], ref, scale, f"ns={ns}")


def test_fr_operator_limits():
    """The C ABI rejects operators beyond 256 points (no GPU needed)."""
    from paper_2003_02633_b200 import _native

    lib = _native.load()
    assert lib.vc3_fr_operator_floats(256) > 0
    assert lib.vc3_fr_operator_floats(257) == -1 and lib.vc3_fr_operator_floats(0) == -1
    assert lib.vc3_fr_divergence_f32(None, None, None, 1, 1, 1, 125, None) == -2


PAIR_SCRIPT = """
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
from paper_2003_02633_b200 import codec, fr
out = {{}}
for k, n_elem, n_vars in ((4, 1000, 5), (1, 37, 2), (2, 300, 3), (5, 260, 1)):
    ns = (k + 1) ** 3
    g = torch.Generator(device="cuda").manual_seed(k)
    F = torch.rand((ns, n_vars, n_elem, 3), device="cuda", generator=g) * 2 - 1
    words = codec.compress(F.reshape(-1, 3)).reshape(ns, n_vars, n_elem)
    op = fr.Operator(fr.divergence_operator(k))
    out[k] = (fr.flux_divergence(words, op).cpu().numpy(), fr.flux_divergence_f32(F, op).cpu().numpy())
np.savez({path!r}, **{{f"c{{k}}": v[0] for k, v in out.items()}}, **{{f"f{{k}}": v[1] for k, v in out.items()}})
print("ok")
"""


@pytest.mark.gpu
def test_fr_pair_kernel_matches(tmp_path):
    """The opt-in CTA-pair kernel (tcgen05 cta_group::2, VC3_FR_PAIR=1) gives
    the single-CTA kernel's results to the 3xTF32 accuracy (both paths
    accumulate the same products in the same order per output)."""
    import os
    import subprocess
    import sys

    root = str(Path(__file__).resolve().parents[1])
    res = {}
    for pair in ("0", "1"):
        path = str(tmp_path / f"fr{pair}.npz")
        env = dict(os.environ, VC3_FR_PAIR=pair)
        r = subprocess.run([sys.executable, "-c", PAIR_SCRIPT.format(root=root, path=path)], env=env,
                           capture_output=True, text=True, timeout=300)
        assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout + r.stderr
        res[pair] = np.load(path)
    for key in res["0"].files:
        a, b = res["0"][key], res["1"][key]
        scale = np.abs(a).max() + 1e-30
        assert np.abs(a - b).max() <= 2.0 ** -16 * scale, key
