"""Host-side pieces of the studies (no GPU): the Smith variable-bin rule and
the report envelope (analysis.py:420-443, 489-500)."""

import pytest

from paper_2003_02633_b200 import DomainError, analysis
from paper_2003_02633_b200.layout import DEFAULT_LAYOUT, DEFAULT_POLICY


def test_smith_theta_bins_matches_reference(golden):
    cases = ((0.3, 64, 0.05), (1.5, 1000, 0.01), (2.9, 131071, 1e-4), (1.0, 8, 0.5))
    got = [analysis.smith_theta_bins(*c) for c in cases]
    assert got == list(golden["smith_bins"])


@pytest.mark.parametrize("args", [(0.0, 64, 0.1), (3.2, 64, 0.1), (1.0, 64, 0.0),
                                  (1.0, 64, -1.0), (1.0, 8, 1e-9)])
def test_smith_theta_bins_domain_errors(args):
    with pytest.raises(DomainError):
        analysis.smith_theta_bins(*args)


def test_report_envelope():
    dom = analysis.SampleDomain("shell", 10, 4, 0.5, 2.0)
    doc = analysis.report(dom, DEFAULT_LAYOUT, DEFAULT_POLICY, extra=1)
    assert doc == {"layout": str(DEFAULT_LAYOUT), "policy": DEFAULT_POLICY.spec(),
                   "domain": "shell:0.5:2", "seed": 4, "count": 10, "extra": 1}


def test_criterion_4b_joint_coding_exact():
    """Acceptance 4b (pkg/tests/test_acceptance.py): exhaustive p = 8 joint round trip."""
    import numpy as np

    cfg = analysis.SplitConfig(8, 11)
    nt, nph = np.meshgrid(np.arange(cfg.n_theta_max + 1), np.arange(cfg.n_phi_max + 1))
    joint = analysis.joint_encode(nt.ravel(), nph.ravel(), cfg)
    nt2, nph2 = analysis.joint_decode(joint, cfg)
    assert joint.max() < 256 and np.array_equal(nt2, nt.ravel()) and np.array_equal(nph2, nph.ravel())


def test_error_metric_restatement_properties():
    """oracle/vc3_stats.py (the CPU restatement of the K6 metrics)."""
    import numpy as np
    import vc3_stats as st

    v = np.array([[1, 0, 0], [0, 2, 0], [3, 4, 0], [0, 0, 0]], np.float32)
    same = st.errors(v, v, st.ANGULAR)
    assert np.array_equal(same, np.zeros(4))
    assert np.allclose(st.errors(v, 2 * v, st.ANGULAR), 0.0)
    orth = np.array([[0, 1, 0], [1, 0, 0], [-4, 3, 0], [1, 1, 1]], np.float32)
    assert np.allclose(st.errors(v, orth, st.ANGULAR)[:3], np.pi / 2)
    assert np.allclose(st.errors(v, 2 * v, st.REL_MAGNITUDE), [1, 1, 1, 0])
    assert np.allclose(st.errors(v, 2 * v, st.L2), [1, 2, 5, 0])
    assert np.allclose(st.errors(v, 2 * v, st.L2_NORMALISED), [1, 1, 1, 0])
    m = st.chunk_moments(np.tile(v, (5, 1)), np.tile(2 * v, (5, 1)), st.L2, 8)
    assert m.shape == (3, 4) and m[:, 0].tolist() == [8, 8, 4]


def test_error_metric_names():
    with pytest.raises(ValueError):
        analysis._kind(False, "cosine")
    assert analysis._kind(True, "l2") == 1 and analysis._kind(True, "angular") == 2
