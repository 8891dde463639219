"""Run the reference's own test suite (pkg/tests, fetched by ``sync.py``)
unmodified against the B200 package: ``lbvh`` resolves to ``shim/lbvh``,
which aliases every ``lbvh.*`` module to ``paper_1908_11807_b200``.  Every
test here needs the GPU (the package has no CPU path)."""

import os
import sys

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
SHIM = os.path.join(HERE, "shim")
for p in (SHIM, ROOT):
    if p not in sys.path:
        sys.path.insert(0, p)
# subprocesses (test_cli's `python -m lbvh.cli`) see the same shim
os.environ["PYTHONPATH"] = os.pathsep.join(
    [SHIM, ROOT] + [p for p in os.environ.get("PYTHONPATH", "").split(os.pathsep) if p])


def pytest_collection_modifyitems(config, items):
    for item in items:
        if str(item.fspath).startswith(HERE):
            item.add_marker(pytest.mark.gpu)
