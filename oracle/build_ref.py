"""Recipe: install the UNMODIFIED reference package into oracle/_ref (checker only).

The reference (``/root/reference/pkg``, pure Python ``voxsplat``) is
pip-installed from a scratch copy (its build writes into the source tree,
and ``/root/reference`` is read-only) with

    python -m pip install --no-index --no-build-isolation --no-deps \
        --target oracle/_ref <copy of /root/reference/pkg>

``--no-deps``: its declared dependency scikit-image is absent from the
offline wheelhouse and is only used by ``fusion.extract_mesh``, off the
path. ``oracle/_ref`` is git-ignored (never committed) and travels to the
GPU box with the working tree, where ``bench.py --impl reference`` runs it
(``oracle/ref_bench.py``). Nothing in the product imports it.

    python oracle/build_ref.py        # no-op when /root/reference is absent
"""

from __future__ import annotations

import shutil
import subprocess
import sys
import tempfile
from pathlib import Path

REF_PKG = Path("/root/reference/pkg")
TARGET = Path(__file__).resolve().parent / "_ref"


def installed() -> bool:
    return (TARGET / "voxsplat" / "__init__.py").exists()


def build(force: bool = False) -> bool:
    """Install (once) the reference into oracle/_ref; False if it is unavailable."""
    if installed() and not force:
        return True
    if not (REF_PKG / "pyproject.toml").exists():
        return False
    with tempfile.TemporaryDirectory() as tmp:
        src = Path(tmp) / "pkg"
        shutil.copytree(REF_PKG, src, ignore=shutil.ignore_patterns("__pycache__", "*.pyc"))
        if TARGET.exists():
            shutil.rmtree(TARGET)
        subprocess.run([sys.executable, "-m", "pip", "install", "--no-index",
                        "--no-build-isolation", "--no-deps", "--quiet", "--target",
                        str(TARGET), str(src)], check=True)
    return installed()


if __name__ == "__main__":
    ok = build(force="--force" in sys.argv)
    print(f"oracle/_ref: {'installed' if ok else 'reference not available'}")
