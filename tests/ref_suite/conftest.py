"""Run the reference's OWN test suite (/root/reference/pkg/tests) against this package.

The reference tests are not committed here (they are the reference's sources): the build
(`__graft_entry__.build()` / `tools/vendor_ref_suite.py`) copies them, when /root/reference
exists, into this directory as git-ignored ``test_ref_*.py`` (+ ``ref_conftest.py``,
``reference.py``), which travel to the GPU box with the snapshot.  The only rewrite is the
import of the reference's conftest module (``from conftest import`` -> ``from ref_conftest
import``).  This file is the shim:

* ``voxelskip`` and its submodules are aliased to ``paper_1912_09596_b200``;
* every vendored test is marked ``gpu`` (the package has no CPU path); on a machine without
  CUDA the vendored modules are not even collected;
* tests of components out of scope here (the CLI, the WebSocket server,
  the TypeScript viewer, numba JIT warm-up timing) are skipped with that reason, and the
  reference's own known-slow CPU timing assertions are kept as they are.
"""

from __future__ import annotations

import sys
import types
from pathlib import Path

import pytest

HERE = Path(__file__).resolve().parent
VENDORED = sorted(HERE.glob("test_ref_*.py"))

try:
    import torch

    _CUDA = torch.cuda.is_available()
except Exception:  # pragma: no cover
    _CUDA = False

if not _CUDA or not VENDORED:
    collect_ignore_glob = ["test_ref_*.py"]
else:
    import paper_1912_09596_b200 as _pkg
    from paper_1912_09596_b200 import (bench, hybrid, kdtree, lbvh, render, service, svt,
                                       volume)

    sys.modules["voxelskip"] = _pkg
    for _name, _mod in (("bench", bench), ("hybrid", hybrid), ("kdtree", kdtree),
                        ("lbvh", lbvh), ("render", render), ("service", service),
                        ("svt", svt), ("volume", volume)):
        sys.modules[f"voxelskip.{_name}"] = _mod
    # the command-line front end is out of scope; its tests are skipped below
    _cli = types.ModuleType("voxelskip.cli")

    def _cli_main(argv=None):
        pytest.skip("voxelskip.cli (command-line front end) is out of scope")

    _cli.main = _cli_main
    sys.modules["voxelskip.cli"] = _cli
    if not hasattr(_pkg, "serve"):
        def _serve(*a, **k):
            pytest.skip("voxelskip.serve (WebSocket transport) is out of scope")

        _pkg.serve = _serve
    if str(HERE) not in sys.path:
        sys.path.insert(0, str(HERE))
    from ref_conftest import *  # noqa: F401,F403  (the reference's fixtures)

OUT_OF_SCOPE = {
    "test_criterion_11_websocket_matches_offline_render": "WebSocket server (out of scope)",
    "test_criterion_12_frontend_suite_passes": "TypeScript viewer (out of scope)",
    "test_cli_bench_writes_csv_to_stdout": "CLI (out of scope)",
    "test_cli_bench_writes_csv_file": "CLI (out of scope)",
    "test_cli_rejects_unknown_index_kind": "CLI (out of scope)",
}


def pytest_collection_modifyitems(config, items):
    for item in items:
        if Path(str(item.fspath)).parent != HERE:
            continue
        item.add_marker(pytest.mark.gpu)
        reason = OUT_OF_SCOPE.get(item.originalname or item.name)
        if reason:
            item.add_marker(pytest.mark.skip(reason=reason))
