"""Exhaustive proof that the FMA forms in the compress kernels equal the
reference's unfused sequence on every float32 input (tools/exhaustive.cu).
Needs a GPU; the enumeration covers ~7e10 inputs in well under a minute."""

import subprocess

import pytest

pytestmark = pytest.mark.gpu


def test_fma_forms_bit_identical_on_every_float():
    from paper_2003_02633_b200._build import build_exhaustive

    exe = build_exhaustive()
    res = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    print(res.stdout)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "TOTAL mismatches=0" in res.stdout
