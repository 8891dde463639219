"""CPU-only tests: host logic, input generators, the C-ABI library surface."""

import ctypes
import os
import re

import numpy as np
import pytest

import paper_1908_11807_b200 as lb
from paper_1908_11807_b200 import _lib, datasets, validation
from paper_1908_11807_b200.geometry import Box, Point, distance_sq, expand, scene_bounds

from conftest import ROOT, has_gpu
from helpers import sha16

HEADER = os.path.join(ROOT, "include", "lbvh_b200.h")


def header_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(lbvh_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    lib = _lib.load_library()
    for name in header_functions():
        assert hasattr(lib, name), name
    assert lib.lbvh_abi_version() == 5
    assert set(_lib.exported_symbols()) == set(header_functions())


def test_library_strerror_and_workspace_sizes():
    lib = _lib.load_library()
    assert lib.lbvh_strerror(0) == b"ok"
    assert lib.lbvh_strerror(4) == b"empty scene"
    for n in (1, 2, 1000, 10**7):
        assert lib.lbvh_build_workspace_bytes(n) >= 20 * n
        assert lib.lbvh_query_workspace_bytes(n) >= 12 * n
        assert lib.lbvh_scan_workspace_bytes(n) > 0


def test_leaf_directory_bits():
    lib = _lib.load_library()
    assert [lib.lbvh_leaf_directory_bits(n) for n in (1, 19, 20, 10**6, 10**7, 10**8, 2**40)] == \
        [0, 0, 3, 18, 21, 24, 24]
    assert lib.lbvh_leaf_directory(None, 0, 3, None, None) == 1


def test_library_rejects_bad_arguments_without_touching_the_device():
    lib = _lib.load_library()
    # empty scene and null pointers are rejected before any launch
    assert lib.lbvh_build(None, None, 0, 30, None, 0, *([None] * 9), 0, 0, None, None, None) == 4
    assert lib.lbvh_build(None, None, 5, 30, None, 0, *([None] * 9), 0, 0, None, None, None) == 1
    assert lib.lbvh_build(None, None, 5, 31, None, 0, *([None] * 9), 0, 0, None, None, None) == 1
    assert lib.lbvh_sort_pairs(None, None, 10, 30, None, 0, None) == 1
    assert lib.lbvh_compact(None, 0, None, None, 1, None, None) == 1


@pytest.mark.skipif(has_gpu(), reason="checks the no-GPU failure mode")
def test_batch_api_fails_loudly_without_gpu():
    with pytest.raises(RuntimeError, match="CUDA device"):
        lb.build(np.zeros((4, 3), np.float32))


def test_dataset_generators_match_reference(digests):
    for key, want in digests["datasets"].items():
        shape, variant, n, seed = key.split(":")
        pts = datasets.generate(datasets.CloudSpec(shape, variant, int(n), int(seed)))
        assert pts.dtype == np.float32 and pts.shape == (int(n), 3)
        assert sha16(pts) == want, key
    assert datasets.default_radius(10) == digests["default_radius_10"]


def test_cloud_file_roundtrip(tmp_path):
    pts = datasets.generate(datasets.CloudSpec("sphere", "hollow", 257, 3))
    for name in ("c.pcl3", "c.csv"):
        p = tmp_path / name
        datasets.save_cloud(p, pts)
        assert np.array_equal(datasets.load_cloud(p), pts)
    (tmp_path / "bad").write_bytes(b"PCL3" + (10).to_bytes(4, "little") + b"\0" * 12)
    with pytest.raises(ValueError, match="truncated"):
        datasets.load_cloud(tmp_path / "bad")


def test_cloudspec_validation():
    with pytest.raises(ValueError):
        datasets.CloudSpec("torus", "filled", 3)
    with pytest.raises(ValueError):
        datasets.CloudSpec.parse("cube", 3)
    assert datasets.CloudSpec.parse("cube:hollow", 5, 2) == datasets.CloudSpec("cube", "hollow", 5, 2)


def test_validation_messages():
    with pytest.raises(ValueError, match=r"must have shape \(n, 3\)"):
        validation.check_points(np.zeros((4, 2)))
    with pytest.raises(ValueError, match="only finite"):
        validation.check_points(np.array([[0, np.nan, 0]]))
    with pytest.raises(ValueError, match="min corner above"):
        validation.check_boxes((np.ones((2, 3)), np.zeros((2, 3))))
    with pytest.raises(ValueError, match=r"\(n, 3\) or \(n, 6\)"):
        validation.check_boxes(np.zeros((3, 4)))
    with pytest.raises(ValueError, match="non-negative"):
        validation.check_radii(-1.0, 3)
    with pytest.raises(ValueError, match=">= 1"):
        validation.check_neighbor_counts(np.array([1, 0]), 2)
    mins, maxs = validation.check_boxes(np.arange(12, dtype=np.float32).reshape(2, 6))
    assert mins.tolist() == [[0, 1, 2], [6, 7, 8]] and maxs.tolist() == [[3, 4, 5], [9, 10, 11]]
    # deferred value checks keep shapes/dtypes but skip the O(n) scan
    arr = validation.check_points(np.array([[0, np.inf, 0]]), device_checks=True)
    assert arr.dtype == np.float32
    assert validation.check_radii(2.0, 7, device_checks=True).ndim == 0


def test_geometry_semantics():
    b = Box(Point(0, 0, 0), Point(1, 1, 1))
    assert distance_sq(Point(1, 1, 1), b) == 0.0
    assert distance_sq(Point(2, 0.5, -1), b) == 2.0
    assert expand(b, Box(Point(-1, 0, 0), Point(0, 3, 0))) == Box(Point(-1, 0, 0), Point(1, 3, 1))
    assert scene_bounds([b]) == b
    with pytest.raises(ValueError, match="empty scene"):
        scene_bounds([])
    with pytest.raises(ValueError):
        Point(float("nan"), 0, 0)
    with pytest.raises(ValueError):
        Box(Point(1, 0, 0), Point(0, 0, 0))


def test_scalar_topology_helpers_match_reference_kats():
    assert lb.common_prefix([0b00100, 0b00101], 0, 1) == 27 + 4
    assert lb.common_prefix([7, 7, 7, 7], 2, 3) == 32 + 31
    assert lb.common_prefix([1, 2], 0, -1) == -1
    assert lb.find_split([0b00100, 0b00101, 0b10000, 0b10001], 0, 3) == 1
    assert lb.find_split([1, 2, 4, 5, 19, 24, 25, 30], 0, 7) == 3
    assert lb.find_split([9, 9, 9, 9], 0, 3) == 1
    assert lb.node_range([0, 1, 6, 7], 0) == (0, 3)
    assert {lb.node_range([0, 1, 6, 7], i) for i in (1, 2)} == {(0, 1), (2, 3)}
    with pytest.raises(ValueError):
        lb.find_split([1, 2], 1, 1)
    with pytest.raises(ValueError):
        lb.node_range([0, 1], 1)
    assert lb.expand_bits_10(0b101) == 0b1000001
    assert lb.sort_by_key([lb.MortonKey(5, 0), lb.MortonKey(3, 1), lb.MortonKey(3, 2),
                           lb.MortonKey(1, 3)]).tolist() == [3, 1, 2, 0]


def test_result_set_validation():
    with pytest.raises(ValueError, match="non-decreasing"):
        lb.ResultSet(np.int64([0, 3, 1]), np.zeros(1, dtype=np.int32))
    with pytest.raises(ValueError, match="total"):
        lb.ResultSet(np.int64([0, 2]), np.zeros(3, dtype=np.int32))
    with pytest.raises(ValueError, match="align"):
        lb.ResultSet(np.int64([0, 1]), np.zeros(1, np.int32), np.zeros(2, np.float32))
    rs = lb.ResultSet(np.int64([0, 2, 2, 5]), np.arange(5, dtype=np.int32))
    assert rs.counts().tolist() == [2, 0, 3] and rs.hits(2).tolist() == [2, 3, 4]
    with pytest.raises(ValueError, match="no distances"):
        rs.hit_distances(0)


def test_query_value_types():
    with pytest.raises(ValueError):
        lb.SpatialQuery(Point(0, 0, 0), -1.0)
    with pytest.raises(ValueError):
        lb.KnnQuery(Point(0, 0, 0), 0)


def test_reference_module_names():
    """``lbvh.oracle`` / ``lbvh.parallel`` exist under the same names."""
    import paper_1908_11807_b200 as lb
    from paper_1908_11807_b200.oracle import brute_knn_batch, brute_radius_sets  # noqa: F401
    from paper_1908_11807_b200.parallel import run_chunked

    assert lb.oracle.brute_knn is lb.brute_knn
    seen = []
    run_chunked(lambda a, b: seen.append((a, b)), 10, 8)
    run_chunked(lambda a, b: seen.append((a, b)), 0, 8)
    assert seen == [(0, 10)]


def header_prototypes():
    """name -> list of C parameter types, parsed from include/lbvh_b200.h."""
    text = re.sub(r"/\*.*?\*/", "", open(HEADER).read(), flags=re.S)
    protos = {}
    for ret, name, params in re.findall(
            r"(int|size_t|uint64_t|const char \*)\s*(lbvh_[a-z0-9_]+)\s*\(([^)]*)\)\s*;", text):
        ps = [p.strip() for p in params.replace("\n", " ").split(",")]
        protos[name] = [] if ps == ["void"] else [re.sub(r"\s*\b\w+$", "", p) for p in ps]
    return protos


_CTYPE = {"int": ctypes.c_int, "int32_t": ctypes.c_int32, "int64_t": ctypes.c_int64,
          "size_t": ctypes.c_size_t, "float": ctypes.c_float, "double": ctypes.c_double,
          "uint64_t": ctypes.c_uint64, "uint32_t": ctypes.c_uint32}


def _same_kind(c_decl: str, ct) -> bool:
    if "*" in c_decl:
        return ct is ctypes.c_void_p or ct is ctypes.c_char_p or issubclass(
            ct, ctypes._Pointer)
    return ctypes.sizeof(ct) == ctypes.sizeof(_CTYPE[c_decl]) and (
        issubclass(ct, ctypes.c_float) == (c_decl == "float")) and (
        issubclass(ct, ctypes.c_double) == (c_decl == "double"))


def test_python_binding_matches_header():
    protos = header_prototypes()
    assert len(protos) == len(header_functions())
    for name, (argtypes, _) in _lib._SIGS.items():
        assert name in protos, name
        assert len(argtypes) == len(protos[name]), (name, len(argtypes), protos[name])
        for c_decl, ct in zip(protos[name], argtypes):
            assert _same_kind(c_decl, ct), (name, c_decl, ct)


def test_integration_stub_matches_header():
    """The ctypes stub INTEGRATION.md tells a reference maintainer to add:
    executed against the built library, every argtypes list it declares must
    match the header prototype parameter for parameter."""
    md = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    block = next(b for b in re.findall(r"```python\n(.*?)```", md, flags=re.S)
                 if "lbvh_build.argtypes" in b)
    block = block.replace("import cupy as cp\n", "cp = None\n").replace(
        '"liblbvh_b200.so"', repr(_lib.LIB_PATH))
    ns = {}
    exec(compile(block, "INTEGRATION.md", "exec"), ns)  # runs the ABI version assert
    stub_lib = ns["_lib"]
    protos = header_prototypes()
    declared = re.findall(r"_lib\.(lbvh_[a-z0-9_]+)\.argtypes", block)
    assert {"lbvh_build", "lbvh_knn", "lbvh_finish_rows"} <= set(declared)
    for name in declared:
        argtypes = getattr(stub_lib, name).argtypes
        assert len(argtypes) == len(protos[name]), (name, len(argtypes), protos[name])
        for c_decl, ct in zip(protos[name], argtypes):
            assert _same_kind(c_decl, ct), (name, c_decl, ct)
    # the stub's tree struct is the header's
    fields = [f for f, _ in ns["LbvhTree"]._fields_]
    assert fields == [f for f, _ in _lib.CTree._fields_]
