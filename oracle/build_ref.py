"""Recipe for oracle/_ref/: the reference package itself, as test and
baseline infrastructure — TEST INFRASTRUCTURE ONLY, never imported by the
product package.

The reference (/root/reference/pkg, `relab`) is pure Python + numpy, so
"building" it is an offline pip install of its own pyproject (setuptools,
--no-index, --no-deps: numpy is already in the image) into
oracle/_ref/site, from a scratch copy (the reference tree is read-only),
plus a copy of its test directory as the package oracle/_ref/relab_tests
so its own tests can run against the B200 operators (tests/
test_gpu_reference_suite.py, through oracle/ref_plugin.py). Nothing here is
committed: oracle/_ref/ is git-ignored (build output, like the .so) and
travels to the GPU box with the working tree, where /root/reference does not
exist. Run by __graft_entry__.build() when /root/reference is present.

    python oracle/build_ref.py [--force]
"""

from __future__ import annotations

import shutil
import subprocess
import sys
import tempfile
from pathlib import Path

REF_PKG = Path("/root/reference/pkg")
OUT = Path(__file__).resolve().parent / "_ref"
SITE = OUT / "site"
TESTS = OUT / "relab_tests"


def available() -> bool:
    return (SITE / "relab" / "tensorpath.py").exists()


def site_path() -> Path:
    return SITE


def build(force: bool = False) -> bool:
    """Install the reference into oracle/_ref. Returns True if it is there."""
    if available() and TESTS.exists() and not force:
        return True
    if not (REF_PKG / "pyproject.toml").exists():
        return available()
    shutil.rmtree(OUT, ignore_errors=True)
    OUT.mkdir(parents=True)
    with tempfile.TemporaryDirectory() as tmp:
        src = Path(tmp) / "pkg"
        shutil.copytree(REF_PKG, src, ignore=shutil.ignore_patterns("__pycache__", "*.pyc", "*.egg-info", "build"))
        subprocess.run([sys.executable, "-m", "pip", "install", "--quiet", "--no-index", "--no-build-isolation",
                        "--no-deps", "--target", str(SITE), str(src)], check=True)
    shutil.copytree(REF_PKG / "tests", TESTS, ignore=shutil.ignore_patterns("__pycache__", "*.pyc"))
    (OUT / "README").write_text("Built by oracle/build_ref.py from /root/reference/pkg (git-ignored build output).\n")
    return available()


if __name__ == "__main__":
    ok = build(force="--force" in sys.argv)
    print(f"oracle/_ref: {'ok' if ok else 'unavailable'} ({SITE})")
