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
