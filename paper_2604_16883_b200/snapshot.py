"""SNKT tensor files (tensor.hpp:86-96) through the library's host C++:
the reference's on-disk format for K/V dumps and cache snapshots (SURVEY.md
§8 f2).  Snapshot save/load live on KvCache (save_snapshot,
load_snapshot, load_snapshot_into)."""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._abi import check, lib


def snkt_file_size(dims) -> int:
    d = np.ascontiguousarray(dims, dtype=np.uint64)
    return int(lib().sinkr_snkt_file_size(d.ctypes.data, C.c_size_t(d.size)))


def write_tensor(path, data) -> None:
    """write_tensor (tensor.cpp:84-99): f32 row-major payload, shape = data.shape."""
    a = np.ascontiguousarray(data, dtype=np.float32)
    dims = np.ascontiguousarray(a.shape, dtype=np.uint64)
    check(lib().sinkr_write_tensor(str(path).encode(), dims.ctypes.data, C.c_size_t(dims.size),
                                   a.ctypes.data))


def read_tensor(path) -> np.ndarray:
    """read_tensor (tensor.cpp:101-140) with the reference's parse errors."""
    dims = np.zeros(64, dtype=np.uint64)
    nd = C.c_size_t()
    check(lib().sinkr_read_tensor(str(path).encode(), dims.ctypes.data, C.byref(nd), None,
                                  C.c_size_t(0)))
    shape = tuple(int(x) for x in dims[:nd.value])
    out = np.zeros(shape, dtype=np.float32)
    check(lib().sinkr_read_tensor(str(path).encode(), dims.ctypes.data, C.byref(nd),
                                  out.ctypes.data, C.c_size_t(out.size)))
    return out
