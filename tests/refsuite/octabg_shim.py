"""pytest plugin: run the reference's OWN test files against this package.

Installs ``octabg`` (and ``octabg.errors/octree/model/detect/evaluation/
frame_io``) in ``sys.modules`` as aliases of ``paper_1412_1945_b200`` before the
reference tests are collected, so ``from octabg import ...`` in
``/root/reference/pkg/tests/*.py`` binds this package's classes and functions.
Only the two reference modules that are out of scope for the drop-in
(the synthetic-scene generator ``synth.py`` and the CLI
``cli.py``) are loaded from the installed, unmodified reference
(``baseline/_ref/octabg``); they import everything else through the alias, so
``octabg.cli.main`` trains and detects with the CUDA path.

Test infrastructure only: the reference files are staged, git-ignored, by
``tools/stage_reference.py`` into ``baseline/_ref_tests`` (they are never
committed) and travel to the GPU box with the snapshot.
"""

from __future__ import annotations

import importlib.util
import os
import sys
import types

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
REF_PKG = os.path.join(REPO, "baseline", "_ref", "octabg")


def _install() -> None:
    if REPO not in sys.path:
        sys.path.insert(0, REPO)
    import paper_1412_1945_b200 as obg
    from paper_1412_1945_b200 import detect, errors, evaluation, frame_io, model, octree

    pkg = types.ModuleType("octabg")
    pkg.__path__ = []          # a package, so ``import octabg.x`` resolves via sys.modules
    pkg.__file__ = obg.__file__
    for name in dir(obg):
        if not name.startswith("__") or name == "__version__":
            setattr(pkg, name, getattr(obg, name))
    sys.modules["octabg"] = pkg
    for sub, mod in (("errors", errors), ("octree", octree), ("model", model),
                     ("detect", detect), ("evaluation", evaluation), ("frame_io", frame_io)):
        sys.modules["octabg." + sub] = mod
        setattr(pkg, sub, mod)
    # out-of-scope reference modules, unmodified, importing the drop-in through the alias
    for sub in ("synth", "cli"):
        path = os.path.join(REF_PKG, sub + ".py")
        spec = importlib.util.spec_from_file_location("octabg." + sub, path)
        mod = importlib.util.module_from_spec(spec)
        sys.modules["octabg." + sub] = mod
        spec.loader.exec_module(mod)
        setattr(pkg, sub, mod)
    for name in ("SCENARIOS", "BoxSpec", "SyntheticParams", "generate_synthetic"):
        setattr(pkg, name, getattr(sys.modules["octabg.synth"], name))


def pytest_configure(config):
    _install()
