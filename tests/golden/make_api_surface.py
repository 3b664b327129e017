"""Record the reference package's public API surface (names and parameter
lists per module) as tests/golden/api_surface.json.  Run in the container
that has /root/reference:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_api_surface.py
"""

import importlib
import inspect
import json
from pathlib import Path

MODULES = ["", ".codec", ".analysis", ".bench", ".stream", ".cli", ".layout", ".errors"]


def main():
    out = {}
    for m in MODULES:
        mod = importlib.import_module("vc3" + m)
        entries = {}
        for name in sorted(dir(mod)):
            if name.startswith("_"):
                continue
            obj = getattr(mod, name)
            if inspect.ismodule(obj) or type(obj).__name__ == "_Feature":
                continue  # imported modules, `from __future__ import annotations`
            if callable(obj) and not getattr(obj, "__module__", "").startswith("vc3"):
                continue  # third-party helpers imported into the namespace (np, Path, field, ...)
            params = None
            if inspect.isfunction(obj):
                params = list(inspect.signature(obj).parameters)
            entries[name] = params
        out["vc3" + m] = entries
    Path(__file__).with_name("api_surface.json").write_text(json.dumps(out, indent=1, sort_keys=True))
    print(sum(len(v) for v in out.values()), "names")


if __name__ == "__main__":
    main()
