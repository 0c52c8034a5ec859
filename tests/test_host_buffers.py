"""Host-side store allocation (``_native.host_empty``): large run outputs are
backed by a huge-page-advised anonymous mapping and must behave exactly like
``np.empty`` arrays for every consumer (writes, slicing, pickling, ctypes)."""

import pickle

import numpy as np

from paper_1908_03869_b200 import _native as nat


def test_small_store_is_plain_ndarray():
    a = nat.host_empty((4, 3, 2))
    assert a.shape == (4, 3, 2) and a.dtype == np.float64 and a.flags.writeable
    assert a.base is None


def test_large_store_is_writable_contiguous_and_outlives_views():
    shape = (nat.HUGE_STORE_BYTES // (8 * 64) + 1, 8, 8)
    a = nat.host_empty(shape)
    assert a.shape == shape and a.dtype == np.float64
    assert a.flags.writeable and a.flags.c_contiguous
    assert a.ctypes.data % 4096 == 0
    a[:] = 2.5
    view = a[1:3]
    del a
    assert float(view.sum()) == 2.5 * view.size
    back = pickle.loads(pickle.dumps(view))
    np.testing.assert_array_equal(back, view)


def test_int_dtype():
    a = nat.host_empty((nat.HUGE_STORE_BYTES // 8,), np.int64)
    a[-1] = 7
    assert a.dtype == np.int64 and a[-1] == 7


def test_large_store_mapping_recycled_only_after_last_view(monkeypatch):
    import gc
    monkeypatch.setenv("SDEB200_HOST_POOL_MB", "1024")
    shape = (nat.HUGE_STORE_BYTES // 8 + 512,)
    a = nat.host_empty(shape)
    addr = a.ctypes.data
    a[:] = 3.0
    view = a[10:20]
    del a
    gc.collect()
    b = nat.host_empty(shape)  # the first mapping is still referenced by `view`
    b_addr = b.ctypes.data
    assert b_addr != addr and float(view.sum()) == 30.0
    del view, b
    gc.collect()
    c = nat.host_empty(shape)  # a released mapping of this size is reused
    assert c.ctypes.data in (addr, b_addr)
    del c
    gc.collect()


def test_pool_disabled(monkeypatch):
    import gc
    monkeypatch.setenv("SDEB200_HOST_POOL_MB", "0")
    a = nat.host_empty((nat.HUGE_STORE_BYTES // 8,))
    a[-1] = 1.0
    del a
    gc.collect()
    assert nat._pool_bytes <= 1024 << 20
