"""Reference module name ``lbvh.parallel`` (pkg/src/lbvh/parallel.py:21): the
host thread-pool chunking of the numba kernels.

On the GPU every batch is one grid launch, so the ``threads`` arguments of the
public API are accepted and ignored; ``run_chunked`` keeps the helper's
contract -- ``fn(start, end)`` covers ``[0, n_items)`` and chunk boundaries
never change results -- with a single inline call.
"""

from __future__ import annotations

from typing import Callable

__all__ = ["run_chunked"]


def run_chunked(fn: Callable[[int, int], None], n_items: int, threads: int = 1) -> None:
    if n_items > 0:
        fn(0, n_items)
