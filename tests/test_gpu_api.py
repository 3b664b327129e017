"""C-ABI hygiene on the device (API items).  Needs a B200.

* the first ever operation for a layout can run inside a caller's CUDA-graph
  capture (the decode tables are built on a private stream in relaxed capture
  mode) and the graph replays bit-identically;
* vc3_prepare_layout builds the tables ahead;
* vc3_error_stats_ws (caller workspace) equals vc3_error_stats;
* magnitude_event_counts on device input raises NonFiniteInput like the host
  path.
"""

import subprocess
import sys
import textwrap
from pathlib import Path

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]

CAPTURE_FIRST_CALL = textwrap.dedent("""
    import sys, numpy as np, torch
    sys.path.insert(0, {root!r})
    import paper_2003_02633_b200 as vc3b
    from paper_2003_02633_b200 import _native
    from paper_2003_02633_b200.layout import BitLayout
    lib = _native.load()
    lay = BitLayout(0, 7, 22, 16, 19, 80)          # a table layout nothing has used yet
    pol = vc3b.ALL_SINGLE_POLICY
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(3)
    n = 100003
    va = torch.rand((n, 3), device=dev, generator=g) * 2 - 1
    vb = torch.rand((n, 3), device=dev, generator=g) * 2 - 1
    # the inputs come from a different layout's compress so that the add's
    # tables (this layout's) are really built inside the capture
    a = torch.randint(0, 2**62, (n,), device=dev, dtype=torch.int64).view(torch.uint64)
    b = torch.randint(0, 2**62, (n,), device=dev, dtype=torch.int64).view(torch.uint64)
    outs = {{}}
    for mode, flags in (("exact", 0), ("contract", 1)):
        c = torch.empty_like(a)
        s = torch.cuda.Stream()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            with torch.cuda.graph(graph, stream=s):
                rc = lib.vc3_add_compressed_ex(a.data_ptr(), b.data_ptr(), c.data_ptr(), n,
                                               _native.c_layout(lay), pol.mask, flags, s.cuda_stream)
        assert rc == 0, rc
        c.zero_()
        graph.replay()
        torch.cuda.synchronize()
        eager = vc3b.add_compressed(a, b, lay, pol, mode=mode)
        torch.cuda.synchronize()
        assert torch.equal(c, eager), mode
        outs[mode] = c
    print("ok")
""")


def test_first_call_captured_in_cuda_graph():
    r = subprocess.run([sys.executable, "-c", CAPTURE_FIRST_CALL.format(root=str(ROOT))],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout + r.stderr


def test_prepare_layout_then_decode_tolerance(vc3b, cuda):
    from paper_2003_02633_b200 import _native
    from paper_2003_02633_b200.layout import BitLayout
    import ctypes

    lib = _native.load()
    lay = BitLayout(0, 7, 22, 17, 18, 80)
    assert lib.vc3_prepare_layout(_native.c_layout(lay), 0) == 0
    tol = ctypes.c_double()
    assert lib.vc3_decode_tolerance(_native.c_layout(lay), ctypes.byref(tol)) == 0
    # measured on the host over every index: a few 2^-49 (decode_tolerance)
    assert 2.0 ** -50 < tol.value < 2.0 ** -45
    assert lib.vc3_prepare_layout(_native.c_layout(lay), 7) == _native.VC3_ERR_ARG


def test_error_stats_workspace_matches(vc3b, cuda):
    import ctypes

    from paper_2003_02633_b200 import _native

    lib = _native.load()
    g = torch.Generator(device=cuda).manual_seed(5)
    n, chunk = 300_001, 1 << 16
    v = torch.rand((n, 3), device=cuda, generator=g)
    vh = v + 1e-6 * torch.rand((n, 3), device=cuda, generator=g)
    nch = (n + chunk - 1) // chunk
    a = torch.empty(4 * nch, dtype=torch.float64, device=cuda)
    b = torch.empty_like(a)
    s = torch.cuda.current_stream().cuda_stream
    assert lib.vc3_error_stats(v.data_ptr(), vh.data_ptr(), n, 1, chunk, a.data_ptr(), s) == 0
    nbytes = ctypes.c_uint64()
    assert lib.vc3_error_stats_workspace(n, chunk, ctypes.byref(nbytes)) == 0
    work = torch.empty(nbytes.value, dtype=torch.uint8, device=cuda)
    assert lib.vc3_error_stats_ws(v.data_ptr(), vh.data_ptr(), n, 1, chunk, b.data_ptr(),
                                  work.data_ptr(), nbytes.value, s) == 0
    assert lib.vc3_error_stats_ws(v.data_ptr(), vh.data_ptr(), n, 1, chunk, b.data_ptr(),
                                  work.data_ptr(), nbytes.value - 1, s) == _native.VC3_ERR_ARG
    torch.cuda.synchronize()
    assert torch.equal(a, b)


def test_magnitude_events_device_nonfinite_raises(vc3b, cuda):
    v = torch.ones((1000, 3), device=cuda)
    v[17, 1] = float("nan")
    v[400, 2] = float("inf")
    with pytest.raises(vc3b.NonFiniteInput):
        vc3b.magnitude_event_counts(v)
    v[17, 1] = 1.0
    v[400, 2] = 1.0
    assert vc3b.magnitude_event_counts(v) == (0, 0)
