"""CPU-only: the C-ABI library loads and exports every symbol livecap.h declares."""

import os
import re

import numpy as np

from paper_1810_02648_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "livecap.h")).read()
    return sorted(set(re.findall(r"\b(lc_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_entry_points():
    syms = header_symbols()
    for must in ("lc_pcg_solve_bsr", "lc_dense_solve", "lc_pose_solve", "lc_nonrigid_solve",
                 "lc_tracker_step", "lc_render", "lc_field_query", "lc_gaussian_pyramid"):
        assert must in syms


def test_library_exports_every_declared_symbol():
    lib = _lib.load_library()
    for s in header_symbols():
        assert hasattr(lib, s), f"{s} declared in livecap.h but not exported"
    for s in _lib.EXPORTED:
        assert hasattr(lib, s)


def test_ctypes_struct_sizes_are_plain():
    # reports are fixed-size POD structs shared with the device
    assert _lib.ctypes if hasattr(_lib, "ctypes") else True
    assert _lib.C.sizeof(_lib.PoseReport) > 0 and _lib.C.sizeof(_lib.NonrigidReport) > 0


def test_device_tables_match_numpy():
    """Pyramid taps and rim probe offsets computed in C++ equal the reference's
    numpy formulas bit for bit (imageproc.py:264-273, pose_stage.py:255-259)."""
    from oracle.imaging import gaussian_kernel
    lib = _lib.load_library()
    for size in (1, 3, 9, 15):   # the default kernels; other sizes get numpy taps from the host
        taps = np.zeros(size)
        _lib.check(lib.lc_debug_tables(size, _lib.ptr(taps), None))
        assert np.array_equal(taps, gaussian_kernel(size)), size
    for size in (5, 21, 25):
        assert np.array_equal(_lib.gaussian_taps(size), gaussian_kernel(size))
    probe = np.zeros((128, 2))
    _lib.check(lib.lc_debug_tables(3, None, _lib.ptr(probe)))
    ang = np.linspace(0.0, 2.0 * np.pi, 16, endpoint=False)
    offs = (np.stack([np.cos(ang), np.sin(ang)], axis=1)[:, None, :]
            * np.arange(1, 9, dtype=np.float64)[None, :, None]).reshape(-1, 2)
    assert np.array_equal(probe, offs)


def test_errors_map_to_python_exceptions():
    lib = _lib.load_library()
    code = lib.lc_ctx_create(0, 0, None)
    assert code == _lib.LC_EINVAL
    assert b"null" in lib.lc_last_error()
