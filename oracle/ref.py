"""Import the unmodified reference package ``negflow`` (test infrastructure only).

Looks in oracle/_ref/negflow.zip (bytecode staged by oracle/make_ref.py; present on the GPU box)
and then in /root/reference/pkg/src (the build container).  Only tests/,
__graft_entry__.smoke() and bench.py's reference arm / cpu_baseline leg may
call this; the product path never does.
"""

from __future__ import annotations

import importlib
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CANDIDATES = (os.path.join(HERE, "_ref", "negflow.zip"), "/root/reference/pkg/src")


def ref_path() -> str | None:
    """sys.path entry holding the reference: the staged bytecode archive, else the source tree."""
    for path in CANDIDATES:
        if path.endswith(".zip") and os.path.isfile(path):
            return path
        if os.path.isfile(os.path.join(path, "negflow", "sse.py")):
            return path
    return None


def import_negflow():
    """The reference package (its submodules sse, distsim, gf, device, params imported)."""
    path = ref_path()
    if path is None:
        raise ImportError("reference negflow not found: run `python oracle/make_ref.py` in the build container")
    if path not in sys.path:
        sys.path.insert(0, path)
    mod = importlib.import_module("negflow")
    for sub in ("sse", "distsim", "gf", "device", "params", "cli", "flops"):
        importlib.import_module(f"negflow.{sub}")
    return mod
