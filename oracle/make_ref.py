"""Test infrastructure (never imported by the product): copy the reference
package and its own test-suite into oracle/_ref so the drop-in integration
tests can run the REAL reference on the GPU box.

The reference is pure Python/numpy (/root/reference/pkg/src/neosim), so
there is nothing to compile; its sources are copied verbatim, out of
history (oracle/_ref/ is git-ignored) but inside the repo snapshot that
gpurun ships to the box, where /root/reference does not exist.  The copy
is refreshed by __graft_entry__.build() whenever /root/reference is present.

    oracle/_ref/neosim/   the reference package (imported by tests/ only)
    oracle/_ref/tests/    pkg/tests (run by tests/test_gpu_reference_suite.py
                          with dropin.install(neosim) applied)
"""
from __future__ import annotations

import shutil
from pathlib import Path

SRC = Path("/root/reference/pkg")
DST = Path(__file__).resolve().parent / "_ref"


def build() -> Path | None:
    """Refresh oracle/_ref from /root/reference (no-op when it is absent)."""
    if not (SRC / "src" / "neosim").is_dir():
        return DST if (DST / "neosim").is_dir() else None
    ignore = shutil.ignore_patterns("__pycache__", "*.pyc", ".pytest_cache", ".hypothesis")
    for sub, dst in ((SRC / "src" / "neosim", DST / "neosim"), (SRC / "tests", DST / "tests")):
        if dst.exists():
            shutil.rmtree(dst)
        shutil.copytree(sub, dst, ignore=ignore)
    return DST


if __name__ == "__main__":
    print(build())
