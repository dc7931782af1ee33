"""Build the UNMODIFIED reference package into oracle/_ref/ (test infrastructure).

The reference ``negflow`` (/root/reference/pkg/src/negflow) is pure Python
(numpy / scipy / sympy), so its build output is CPython bytecode: every
module is compiled, where it lies under /root/reference, into a sourceless
package

    python oracle/make_ref.py        # also run by __graft_entry__.build()

-> oracle/_ref/negflow.zip holding negflow/<module>.pyc (imported by CPython's
zipimport, which loads sourceless bytecode; the image's Python 3.12 on both
sides) plus oracle/_ref/SOURCE.json (sha256 of every source file compiled).  No reference source is copied into the repo.
oracle/_ref/ is git-ignored but travels to the GPU box with the gpurun
snapshot, where /root/reference does not exist: there it is the reference
arm of bench.py (``--impl reference``), the cpu_baseline leg and the checker
of the GPU compat tests (tests/test_gpu_reference.py).  Nothing on the
product path imports it.
"""

from __future__ import annotations

import hashlib
import json
import os
import py_compile
import shutil
import sys
import tempfile
import zipfile

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = "/root/reference/pkg/src/negflow"
DST = os.path.join(HERE, "_ref", "negflow.zip")
MANIFEST = os.path.join(HERE, "_ref", "SOURCE.json")


def sha256(path: str) -> str:
    with open(path, "rb") as fh:
        return hashlib.sha256(fh.read()).hexdigest()


def stage(src: str = SRC) -> str | None:
    """Compile the reference package into oracle/_ref; None when the reference is absent."""
    if not os.path.isdir(src):
        return None
    os.makedirs(os.path.dirname(DST), exist_ok=True)
    files = sorted(f for f in os.listdir(src) if f.endswith(".py"))
    tmp = DST + ".tmp"
    with tempfile.TemporaryDirectory() as work, zipfile.ZipFile(tmp, "w", zipfile.ZIP_DEFLATED) as zf:
        for f in files:
            pyc = os.path.join(work, f[:-3] + ".pyc")
            py_compile.compile(os.path.join(src, f), cfile=pyc, doraise=True,
                               invalidation_mode=py_compile.PycInvalidationMode.UNCHECKED_HASH)
            zf.write(pyc, arcname=f"negflow/{f[:-3]}.pyc")
    os.replace(tmp, DST)
    manifest = {"source": src, "python": sys.version.split()[0],
                "files": {f: sha256(os.path.join(src, f)) for f in files}}
    with open(MANIFEST, "w") as fh:
        json.dump(manifest, fh, indent=1)
    return DST


if __name__ == "__main__":
    out = stage(sys.argv[1] if len(sys.argv) > 1 else SRC)
    print(out or f"{SRC} not present: nothing staged")
