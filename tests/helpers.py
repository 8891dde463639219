"""Shared comparators for the parity tests."""

import hashlib

import numpy as np

TREE_FIELDS = ("node_mins", "node_maxs", "left", "right", "leaf_obj", "scene_min", "scene_max")


def sha16(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def sorted_concat(offsets, indices):
    offsets = np.asarray(offsets)
    indices = np.asarray(indices)
    out = np.empty_like(indices)
    for q in range(offsets.shape[0] - 1):
        s, e = offsets[q], offsets[q + 1]
        out[s:e] = np.sort(indices[s:e])
    return out


def assert_same_tree(tree, g, prefix):
    for f in TREE_FIELDS:
        got = np.asarray(getattr(tree, f))
        want = g[prefix + f]
        assert got.dtype == want.dtype, (f, got.dtype, want.dtype)
        assert got.shape == want.shape, (f, got.shape, want.shape)
        if f.startswith("scene"):
            assert np.array_equal(got, want), f  # +-0 may differ in sign
        else:
            assert got.tobytes() == want.tobytes(), f"{prefix}{f} differs"


def in_order_leaves(left, right, leaf_obj):
    n = leaf_obj.shape[0]
    if n == 1:
        return [int(leaf_obj[0])]
    out, stack = [], [0]
    while stack:
        node = stack.pop()
        if node >= n - 1:
            out.append(int(leaf_obj[node - (n - 1)]))
        else:
            stack.append(int(right[node]))
            stack.append(int(left[node]))
    return out
