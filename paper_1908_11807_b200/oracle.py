"""Reference module name ``lbvh.oracle`` (pkg/src/lbvh/oracle.py:18-70): the
brute-force neighbour helpers, here the GPU kernels of :mod:`.brute`.

This is part of the drop-in API (the reference's own tests import
``brute_knn_batch`` / ``brute_radius_sets`` from ``lbvh.oracle``); it is not
the repository's CPU test oracle (top-level ``oracle/``), which product code
never imports.
"""

from .brute import brute_knn, brute_knn_batch, brute_radius, brute_radius_sets

__all__ = ["brute_radius", "brute_knn", "brute_radius_sets", "brute_knn_batch"]
