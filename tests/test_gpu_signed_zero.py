"""Zero-field words in the fused operations under every precision policy
(ADVICE r1, medium): a zero field decodes to the reference's (+0, +0, +0).
Theta-double policies quantise atan2(y, x), which sees the sign of a zero y,
so a (-0, -0, +0) decode would move the left-half-plane sums below by half a
turn.  Needs a B200."""
import numpy as np
import pytest
import torch

from conftest import layout_by_name, policy_by_code

pytestmark = pytest.mark.gpu

ALL_CODES = ["SSS", "SSD", "SDS", "SDD", "DSS", "DSD", "DDS", "DDD"]


def _dev(w, cuda):
    return torch.from_numpy(np.ascontiguousarray(w)).to(cuda)


@pytest.mark.parametrize("code", ALL_CODES)
def test_zero_word_plus_left_half_plane(vc3b, oracle, cuda, code):
    from paper_2003_02633_b200 import ops

    lay, pol = layout_by_name("17_18"), policy_by_code(code)
    v = np.array([[-1e-6, 0.0, 1.0], [-3.0, 0.0, 0.5], [-2.0, -0.0, -1.0], [-1.0, 0.0, 0.0],
                  [-5e-3, 0.0, -7.0], [-1e-30, 0.0, 1.0], [-2.5, 1e-9, 0.0], [-2.5, -1e-9, 0.0]],
                 np.float32)
    v = np.tile(v, (16, 1))
    b = oracle.compress(v, lay, pol)
    z = np.zeros_like(b)
    for x, y in ((z, b), (b, z)):
        want = oracle.add_compressed(x, y, lay, pol)
        got = ops.add_compressed(_dev(x, cuda), _dev(y, cuda), lay, pol).cpu().numpy()
        assert np.array_equal(got, want), [hex(int(g)) for g in got[got != want][:4]]
    for alpha in (1.0, -0.5):
        want = oracle.axpy(alpha, z, b, lay, pol)
        got = ops.axpy(alpha, _dev(z, cuda), _dev(b, cuda), lay, pol).cpu().numpy()
        assert np.array_equal(got, want), alpha
    # RK stage with a zero dq and a zero R: q' = q + b * (a * 0 + dt * 0) = q
    q, dq, R = b.copy(), z.copy(), z.copy()
    qd, dqd = _dev(q, cuda), _dev(dq, cuda)
    ops.rk_stage(-0.4178, 0.6, 1e-3, qd, dqd, _dev(R, cuda), lay, pol)
    vq = oracle.decompress(q, lay)
    d_new = np.zeros_like(vq)
    q_new = (vq + np.float32(0.6) * d_new).astype(np.float32)
    assert np.array_equal(qd.cpu().numpy(), oracle.compress(q_new, lay, pol))
    assert np.array_equal(dqd.cpu().numpy(), oracle.compress(d_new, lay, pol))
