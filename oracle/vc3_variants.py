"""CPU restatement of the reference's K7 variant round trips (numpy).

TEST INFRASTRUCTURE ONLY (parity checker; see vc3_oracle.py for who may
import it).  Follows /root/reference/pkg/src/vc3/analysis.py:
  compand_study reconstruction   analysis.py:396-417
  Compander.encode / decode      analysis.py:364-393
  split_sweep reconstruction     analysis.py:309-337
  _quantize_free / joint codes   analysis.py:284-306
with the angles and magnitude codes from the C oracle (ORACLE policy).
Pinned to the reference by tests/test_oracle.py (golden ``cmp_*``/``split_*``).
"""

from __future__ import annotations

import math

import numpy as np

import vc3_oracle

_ORACLE = type("P", (), {"theta_single": False, "phi_single": False, "quant_single": False})()


def _angles_and_rh(v, layout):
    r, th, ph = vc3_oracle.to_spherical(v, _ORACLE)
    rh = vc3_oracle.decode_magnitude(vc3_oracle.encode_magnitude(r, layout), layout)
    return r, th, ph, rh.astype(np.float64)


def compand_encode(psi, n_max, kind, gamma=0.5):
    psi = np.asarray(psi, dtype=np.float64)
    if kind == "uniform":
        raw = psi * n_max
    elif kind == "cosine":
        raw = n_max * (1.0 - np.cos(np.pi * psi)) / 2.0
    else:
        c = math.tanh(gamma)
        raw = (1.0 / (2.0 * c)) * n_max * (np.tanh(gamma * (2.0 * psi - 1.0)) + c)
    return np.clip(np.ceil(np.floor(2.0 * raw) / 2.0).astype(np.int64), 0, n_max)


def compand_decode(n, n_max, kind, gamma=0.5):
    n = np.asarray(n, dtype=np.float64)
    if kind == "uniform":
        return n / n_max
    if kind == "cosine":
        return np.arccos(np.clip(1.0 - 2.0 * n / n_max, -1.0, 1.0)) / np.pi
    c = math.tanh(gamma)
    u = np.clip(n / ((1.0 / (2.0 * c)) * n_max) - c, -c, c)
    return np.clip((np.arctanh(u) / gamma + 1.0) / 2.0, 0.0, 1.0)


def _reconstruct(rh, th2, ph2):
    sp = np.sin(ph2)
    return np.stack([rh * np.cos(th2) * sp, rh * np.sin(th2) * sp, rh * np.cos(ph2)],
                    axis=1).astype(np.float32)


def compand_round_trip(v, layout, kind, gamma=0.5):
    """(n_theta, n_phi, vh) as compand_study computes them."""
    _, th, ph, rh = _angles_and_rh(v, layout)
    ntmax, npmax = layout.n_theta_max, layout.n_phi_max
    nt = compand_encode((th + np.pi) / (2.0 * np.pi), ntmax, kind, gamma)
    nph = compand_encode(ph / np.pi, npmax, kind, gamma)
    th2 = 2.0 * np.pi * compand_decode(nt, ntmax, kind, gamma) - np.pi
    ph2 = np.pi * compand_decode(nph, npmax, kind, gamma)
    return nt, nph, _reconstruct(rh, th2, ph2)


def split_round_trip(v, layout, total_bits, n_phi_max):
    """(joint index, vh) as split_sweep computes them."""
    _, th, ph, rh = _angles_and_rh(v, layout)
    nt_max = (1 << total_bits) // (n_phi_max + 1) - 1
    vt = nt_max / 2.0 + th * (nt_max / (2.0 * np.pi))
    vp = ph * (n_phi_max / np.pi)
    nt = np.clip(np.ceil(np.floor(2.0 * vt) / 2.0).astype(np.int64), 0, nt_max)
    nph = np.clip(np.ceil(np.floor(2.0 * vp) / 2.0).astype(np.int64), 0, n_phi_max)
    joint = nph * (nt_max + 1) + nt
    nt2, nph2 = joint % (nt_max + 1), joint // (nt_max + 1)
    th2 = np.pi * (2.0 * nt2 / nt_max - 1.0)
    ph2 = np.pi * nph2 / n_phi_max
    return joint, _reconstruct(rh, th2, ph2)
