"""The C-ABI library: builds for sm_100a, loads, exports every symbol the
public header declares, and validates arguments before touching a device.
CPU only (no kernel launches)."""

import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "vc3_b200.h"


def header_functions():
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return sorted(set(re.findall(r"\b(vc3_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    from paper_2003_02633_b200 import _native

    lib = _native.load()
    names = header_functions()
    assert len(names) >= 20
    for name in names:
        assert hasattr(lib, name), name
    # the Python signature table covers the header exactly
    assert sorted(_native.SIGNATURES) == names


def test_library_is_sm100a_only():
    from paper_2003_02633_b200 import _native

    out = subprocess.run(["cuobjdump", "--list-elf", str(_native.LIB_PATH)],
                         capture_output=True, text=True, check=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_host_side_validation_without_device():
    from paper_2003_02633_b200 import _native
    from paper_2003_02633_b200.layout import DEFAULT_LAYOUT

    lib = _native.load()
    good = _native.c_layout(DEFAULT_LAYOUT)
    bad = _native.Layout(0, 7, 22, 17, 17, 80)  # sums to 63
    assert lib.vc3_validate_layout(good) == 0
    assert lib.vc3_validate_layout(bad) == _native.VC3_ERR_LAYOUT
    assert lib.vc3_validate_layout(_native.Layout(0, 8, 23, 16, 17, 80)) == _native.VC3_ERR_LAYOUT
    # bad layout / policy / length are rejected before any launch
    assert lib.vc3_compress(None, None, 10, bad, 0, None, None) == _native.VC3_ERR_LAYOUT
    assert lib.vc3_add_compressed(None, None, None, 10, good, 9, None) == _native.VC3_ERR_ARG
    assert lib.vc3_add_compressed(None, None, None, -1, good, 7, None) == _native.VC3_ERR_ARG
    assert lib.vc3_decompress(None, None, 0, good, None) == 0  # empty is a no-op
    assert lib.vc3_add_compressed_host(None, None, None, 0, good, 7, 0) == 0
    assert lib.vc3_status_string(_native.VC3_ERR_NONFINITE) == b"non-finite input"
    assert b"sm_100a" in lib.vc3_version()


def test_status_mapping():
    from paper_2003_02633_b200 import _native, errors

    with pytest.raises(errors.BadLayout):
        _native.check(_native.VC3_ERR_LAYOUT)
    with pytest.raises(errors.NonFiniteInput):
        _native.check(_native.VC3_ERR_NONFINITE)
    with pytest.raises(errors.LengthMismatch):
        _native.check(_native.VC3_ERR_LENGTH)
    with pytest.raises(ValueError):
        _native.check(_native.VC3_ERR_ARG)
    _native.check(0)


def test_no_oracle_on_product_path():
    """The product package never imports or links the oracle."""
    pkg = ROOT / "paper_2003_02633_b200"
    for f in list(pkg.rglob("*.py")) + list(pkg.rglob("*.cu")) + list(pkg.rglob("*.cuh")):
        text = f.read_text()
        assert "vc3_oracle" not in text and "oracle/" not in text, f


def test_python_api_surface_matches_reference():
    """Every public name of the reference package's modules exists here, and
    every reference function's parameters are a prefix of ours (same names,
    same order).  tests/golden/api_surface.json is recorded from the
    reference by tests/golden/make_api_surface.py."""
    import importlib
    import inspect
    import json
    from pathlib import Path

    surface = json.loads((Path(__file__).parent / "golden" / "api_surface.json").read_text())
    problems = []
    for mod_name, entries in surface.items():
        ours = importlib.import_module(mod_name.replace("vc3", "paper_2003_02633_b200", 1))
        for name, params in entries.items():
            if not hasattr(ours, name):
                problems.append(f"{mod_name}.{name} missing")
                continue
            obj = getattr(ours, name)
            if params is not None and inspect.isfunction(obj):
                mine = list(inspect.signature(obj).parameters)
                if mine[: len(params)] != params:
                    problems.append(f"{mod_name}.{name}{tuple(params)} vs ours {tuple(mine)}")
    assert not problems, problems


def test_alias_as_vc3(monkeypatch):
    """``alias_as_vc3`` makes reference-style imports resolve to this package."""
    import importlib
    import sys

    for k in [k for k in sys.modules if k == "vc3" or k.startswith("vc3.")]:
        monkeypatch.delitem(sys.modules, k)
    import paper_2003_02633_b200 as pkg

    pkg.alias_as_vc3()
    try:
        vc3 = importlib.import_module("vc3")
        from vc3 import analysis, codec, stream  # noqa: F401

        assert vc3 is pkg and codec.compress is pkg.compress
        assert stream.HEADER_SIZE == 20 and hasattr(analysis, "error_study")
    finally:
        for k in [k for k in sys.modules if k == "vc3" or k.startswith("vc3.")]:
            del sys.modules[k]
