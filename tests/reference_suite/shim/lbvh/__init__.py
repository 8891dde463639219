"""Import shim: ``lbvh`` (the reference package name) -> paper_1908_11807_b200.

Lets the reference's own test files (``tests/reference_suite/vendored/``) and
``python -m lbvh.cli`` run unmodified against the B200 package.  Every
reference submodule name is aliased to the package's module of the same role
(``lbvh.bench`` is ``harness``), so monkeypatching ``lbvh.traversal`` patches
the real module.
"""

import sys

import paper_1908_11807_b200 as _pkg
from paper_1908_11807_b200 import *  # noqa: F401,F403
from paper_1908_11807_b200 import __all__, __version__  # noqa: F401

from paper_1908_11807_b200 import (  # noqa: E402
    datasets, estimator, geometry, harness, morton, oracle, parallel, traversal, tree,
    validation,
)

_ALIASES = {
    "datasets": datasets, "estimator": estimator, "geometry": geometry, "bench": harness,
    "morton": morton, "oracle": oracle, "parallel": parallel, "traversal": traversal,
    "tree": tree, "validation": validation,
}
for _name, _mod in _ALIASES.items():
    sys.modules[f"{__name__}.{_name}"] = _mod
    globals()[_name] = _mod
del _name, _mod, _pkg
