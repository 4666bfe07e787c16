"""The reference's OWN test files, unmodified, run against this package.

``tests/refsuite/octabg_shim.py`` aliases ``octabg`` -> ``paper_1412_1945_b200``
(the out-of-scope ``octabg.synth`` / ``octabg.cli`` come from the installed
reference and call this package through the alias), then pytest runs
``/root/reference/pkg/tests/*.py`` as staged, git-ignored, in
``baseline/_ref_tests`` by ``tools/stage_reference.py`` (``build()``).  This is
the "switching is an import" claim of INTEGRATION.md, tested.

CPU (``not gpu``): the files that need no CUDA device -- octree serialisation
and properties incl. the hypothesis round trip at its default deadline
(reference ``tests/test_octree.py:238-247``), evaluation, frame I/O.
GPU: every file, build / merge / detect / CLI / acceptance criteria included.
"""

from __future__ import annotations

import os
import subprocess
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_TESTS = os.path.join(REPO, "baseline", "_ref_tests")
REF_PKG = os.path.join(REPO, "baseline", "_ref", "octabg")

ALL_FILES = ["test_octree.py", "test_model.py", "test_detect.py", "test_evaluation.py",
             "test_frame_io.py", "test_cli.py", "test_acceptance.py"]
# tests in the CPU files that call a CUDA entry point (pack_codes runs on the GPU)
CPU_DESELECT = ["test_octree.py::test_pack_codes_matches_scalar"]


def _run(files, deselect=(), timeout=1800):
    if not (os.path.isdir(REF_TESTS) and os.path.isdir(REF_PKG)):
        pytest.skip("reference tests not staged (run tools/stage_reference.py where /root/reference exists)")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([os.path.join(REPO, "tests", "refsuite"), REPO, env.get("PYTHONPATH", "")])
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "octabg_shim", "-p", "no:cacheprovider", "--rootdir", REF_TESTS]
    cmd += [os.path.join(REF_TESTS, f) for f in files]
    for d in deselect:
        cmd += ["--deselect", d]
    r = subprocess.run(cmd, cwd=REF_TESTS, env=env, capture_output=True, text=True, timeout=timeout)
    tail = (r.stdout + r.stderr)[-6000:]
    assert r.returncode == 0, tail
    return tail


def test_reference_suite_cpu_files():
    out = _run(["test_octree.py", "test_evaluation.py", "test_frame_io.py"], CPU_DESELECT)
    assert " passed" in out


@pytest.mark.gpu
@pytest.mark.parametrize("name", ALL_FILES)
def test_reference_suite_gpu(cuda, name):
    out = _run([name])
    assert " passed" in out and "failed" not in out
