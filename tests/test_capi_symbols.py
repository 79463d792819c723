"""The C-ABI library loads and exports every symbol include/tsg.h declares (CPU only; no
compute calls — there is no GPU here), and fails loudly instead of falling back."""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "tsg.h")).read()
    return sorted(set(re.findall(r"\b(tsg_[a-z0-9_]+)\s*\(", text)))


def test_header_and_binding_agree(capi):
    assert sorted(capi.EXPORTS) == declared_symbols()


def test_library_exports_every_declared_symbol(capi):
    L = capi.lib()
    for name in declared_symbols():
        assert hasattr(L, name), name
    assert L.tsg_abi_version() == 1


def test_library_targets_sm100a():
    so = os.path.join(ROOT, "paper_1502_00355_b200", "libtsg.so")
    data = open(so, "rb").read()
    assert b"sm_100a" in data


def test_no_device_is_reported_not_faked(capi):
    if capi.lib().tsg_device_count() > 0:
        pytest.skip("a device is present")
    with pytest.raises(RuntimeError, match="no CUDA device"):
        capi.Context(0)


def test_hilbert_order_is_a_permutation(capi, ts):
    xy, _ = ts.delaunay_arrays(5000, 1)
    order = capi.hilbert_order(xy)
    assert np.array_equal(np.sort(order), np.arange(len(xy)))
    # locality: consecutive slots are spatially close on average
    step = np.linalg.norm(np.diff(xy[order], axis=0), axis=1).mean()
    rand = np.linalg.norm(np.diff(xy, axis=0), axis=1).mean()
    assert step < rand / 10


def test_smooth_without_device_raises(ts):
    if ts.device_count() > 0:
        pytest.skip("a device is present")
    m = ts.generate_grid(5, 5)
    with pytest.raises(RuntimeError, match="no CUDA device"):
        ts.smooth(m)
