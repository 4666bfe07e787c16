"""Stage the reference for the test/bench arms (run by ``__graft_entry__.build``
in the build container, where ``/root/reference`` exists):

* ``baseline/_ref``       -- the unmodified reference package, pip-installed
  (``--no-index --no-deps --target``) from a /tmp copy of ``/root/reference/pkg``;
* ``baseline/_ref_tests`` -- a copy of the reference's own ``pkg/tests``, run
  against this package by ``tests/test_reference_suite.py``.

Both are git-ignored (never committed) and gpurun-included (they travel to the
GPU box, which has no /root/reference).
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
import tempfile

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = "/root/reference/pkg"


def stage(force: bool = False) -> bool:
    if not os.path.isdir(REF):
        return False
    ref_dst = os.path.join(REPO, "baseline", "_ref")
    if force or not os.path.isfile(os.path.join(ref_dst, "octabg", "model.py")):
        with tempfile.TemporaryDirectory() as tmp:
            src = os.path.join(tmp, "pkg")
            shutil.copytree(REF, src)
            subprocess.run([sys.executable, "-m", "pip", "install", "-q", "--no-index",
                            "--no-build-isolation", "--no-deps", "--find-links", "/opt/wheelhouse",
                            "--target", ref_dst, "--upgrade", src], check=True)
    tests_dst = os.path.join(REPO, "baseline", "_ref_tests")
    if os.path.isdir(tests_dst):
        shutil.rmtree(tests_dst)
    shutil.copytree(os.path.join(REF, "tests"), tests_dst,
                    ignore=shutil.ignore_patterns("__pycache__", "*.pyc"))
    return True


if __name__ == "__main__":
    print("staged" if stage(force="--force" in sys.argv) else "no /root/reference here")
