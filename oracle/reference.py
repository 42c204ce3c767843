"""TEST INFRASTRUCTURE — the unmodified reference package (`hetmf`), installed
under oracle/_ref for parity tests and the CPU reference arm only.

Recipe (run by __graft_entry__.build() in the build container, where
/root/reference exists): `pip install --no-index --no-deps --target
oracle/_ref <copy of /root/reference/pkg>` — the reference's own setuptools
build of its own sources, nothing edited.  oracle/_ref is git-ignored (it is
not product source and never enters history) but not gpurun-ignored, so the
installed package travels to the GPU box like the built .so files; nothing
on the box reads /root/reference.

Only tests/, __graft_entry__.smoke() and bench.py's reference / cpu_baseline
legs may import this module.  The product package never does (a not-gpu test
checks that).
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
import tempfile
from pathlib import Path

HERE = Path(__file__).resolve().parent
TARGET = HERE / "_ref"
SOURCE = Path("/root/reference/pkg")


def installed() -> bool:
    return (TARGET / "hetmf" / "__init__.py").exists()


def install(force: bool = False) -> bool:
    """Install the reference into oracle/_ref (no-op when present or when the
    reference tree is absent, e.g. on the GPU box).  Returns installed()."""
    if installed() and not force:
        return True
    if not SOURCE.exists():
        return installed()
    with tempfile.TemporaryDirectory() as tmp:
        src = Path(tmp) / "pkg"          # the reference tree is read-only: build from a copy
        shutil.copytree(SOURCE, src)
        if TARGET.exists():
            shutil.rmtree(TARGET)
        subprocess.run([sys.executable, "-m", "pip", "install", "--quiet", "--no-index",
                        "--no-build-isolation", "--no-deps", "--target", str(TARGET), str(src)],
                       check=True)
    return installed()


def hetmf():
    """Import the installed reference package (numba cache under oracle/_ref)."""
    if not installed():
        raise ImportError("the reference is not installed under oracle/_ref "
                          "(oracle.reference.install() in the build container)")
    os.environ.setdefault("NUMBA_CACHE_DIR", str(TARGET / "numba_cache"))
    if str(TARGET) not in sys.path:
        sys.path.insert(0, str(TARGET))
    import hetmf as ref
    return ref
