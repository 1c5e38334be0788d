"""C-ABI boundary checks that need no GPU: the library loads, exports every
symbol include/ddm.h declares, and its host-only size queries behave."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "ddm.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ddm_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def L():
    from paper_1703_06680_b200 import _build, ddm
    _build.build()
    return ddm.load()


def test_header_declares_the_boundary():
    fns = header_functions()
    for f in ["ddm_match_count", "ddm_match_pairs", "ddm_workspace_bytes", "ddm_sub_index_build",
              "ddm_match_pairs_indexed", "ddm_sort_pairs", "ddm_radix_sort_u64", "ddm_status_string"]:
        assert f in fns


def test_library_exports_every_declared_symbol(L):
    from paper_1703_06680_b200 import ddm
    raw = ctypes.CDLL(ddm.lib_path())
    for f in header_functions():
        assert hasattr(raw, f), f"libddm.so does not export {f}"
    assert sorted(ddm.EXPORTED) == header_functions()


def test_status_strings(L):
    names = [L.ddm_status_string(i).decode() for i in range(7)]
    assert names == ["DDM_OK", "DDM_ERR_INVALID_ARGUMENT", "DDM_ERR_NONFINITE", "DDM_ERR_INVERTED_INTERVAL",
                     "DDM_ERR_CAPACITY", "DDM_ERR_WORKSPACE", "DDM_ERR_CUDA"]


def test_workspace_queries_host_only(L):
    assert L.ddm_workspace_bytes(0, 10, 10, 1) == 0          # d == 0 invalid
    assert L.ddm_workspace_bytes(9, 10, 10, 1) == 0          # d > DDM_MAX_DIMS
    small = L.ddm_workspace_bytes(1, 1000, 1000, 1)
    big = L.ddm_workspace_bytes(1, 10**6, 10**6, 1)
    assert 0 < small < big
    # c3 fits comfortably in one B200 (design budget ~7 GB)
    c3 = L.ddm_workspace_bytes(1, 5 * 10**7, 5 * 10**7, 1)
    assert c3 < 8 * 2**30
    # c5 on one GPU (N = 1e9) stays under the 180 GB HBM
    assert L.ddm_workspace_bytes(1, 5 * 10**8, 5 * 10**8, 1) < 120 * 2**30
    assert L.ddm_sub_index_bytes(3, 1000) > L.ddm_sub_index_bytes(1, 1000)
    assert L.ddm_indexed_workspace_bytes(1, 1000, 1000) > 0
    assert L.ddm_sort_pairs_workspace_bytes(10**6) > 8 * 10**6


def test_build_info(L):
    assert "sm_100a" in L.ddm_build_info().decode()


def test_binding_refuses_cpu_tensors():
    import torch
    from paper_1703_06680_b200 import ddm
    x = torch.zeros((1, 4), dtype=torch.float64)
    with pytest.raises(TypeError):
        ddm.match_count(x, x, x, x)


def test_sort_size_limits_refused_host_only(L):
    """Sorts of more than DDM_MAX_SORT_KEYS keys (the look-back words' 30-bit
    prefixes) are refused with DDM_ERR_INVALID_ARGUMENT before any device
    work (never silently overflowed)."""
    big = 2**30  # DDM_MAX_SORT_KEYS + 1
    fake = 1 << 20  # aligned, never dereferenced: the size check comes first
    assert L.ddm_sort_pairs(fake, big, 10, 10, fake, 2**62, None) == 1
    assert L.ddm_radix_sort_u64(fake, None, fake + 4096, None, big, 0, 64, fake, 2**62, None) == 1
