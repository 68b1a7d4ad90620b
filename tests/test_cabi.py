"""C ABI and code generator, CPU only (no compute calls need a GPU here)."""

import ctypes as C
import re

import numpy as np
import pytest

import fixtures as fx


def _header_symbols():
    import os
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    text = open(os.path.join(root, "include", "cprrtc.h")).read()
    return sorted(set(re.findall(r"CPRRTC_API [^(]*?\b(cprrtc_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    from paper_2505_06791_b200 import _lib
    L = _lib.load()
    syms = _header_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(_lib.EXPORTS)
    assert L.cprrtc_abi_version() == 2


def test_no_gpu_means_loud_failure():
    from paper_2505_06791_b200 import _lib
    if _lib.device_count() > 0:
        pytest.skip("a GPU is visible")
    from paper_2505_06791_b200 import kernels
    from paper_2505_06791_b200.errors import DeviceError
    with pytest.raises(DeviceError):
        kernels.fk_batch(fx.robot("planar2"), np.zeros((1, 2)))


def test_codegen_folds_constants():
    from paper_2505_06791_b200 import _lib
    src = _lib.codegen(fx.robot("arm7").packed)
    assert "#define CP_N 7" in src and "#define CP_S 10" in src and "#define CP_P 7" in src
    assert src.count("cp_sincos(q[") == 7            # one per revolute joint
    assert "T(0.33300000000000002)" in src           # shoulder height folded in
    src8 = _lib.codegen(fx.robot("arm8").packed)
    assert src8.count("cp_sincos(q[") == 7           # the prismatic torso has none
    assert "q[0]" in src8
    dense = _lib.codegen(fx.robot("arm8_dense").packed)
    assert "#define CP_S 36" in dense and "#define CP_P 96" in dense


def test_codegen_rejects_bad_robot():
    from paper_2505_06791_b200 import _lib
    from types import SimpleNamespace
    bad = SimpleNamespace(**{k: getattr(fx.robot("planar2").packed, k) for k in
                             ("jtypes", "axes", "origin_r", "origin_p", "lo", "hi", "sphere_local",
                              "sphere_radius", "pairs")})
    bad.sphere_link = np.array([0, 5], np.int32)
    bad.ee_link = 1
    with pytest.raises(ValueError, match="sphere link"):
        _lib.codegen(bad)


def test_device_source_is_one_translation_unit():
    from paper_2505_06791_b200 import _lib
    src = _lib.device_source(fx.robot("planar2").packed, 16, 0, 0, 0)
    for k in ("cp_plan_kernel", "cp_init_kernel", "cp_check_kernel", "cp_extract_query", "cp_dense_kernel",
              "#define CP_G 16", "struct alignas(128) QueryState"):
        assert k in src
    assert "cp_validate_kernel" in src and "#if CP_PARITY" in src


def test_shared_struct_layout_matches_ctypes():
    from paper_2505_06791_b200 import _lib
    assert C.sizeof(_lib.Result) == 4 * 5 + 4 + 8 + 8 * 12
    assert C.sizeof(_lib.Params) > 0


def test_fast_path_module_loads():
    """The CPython fast path of the single-query plan() (csrc/pyfast.c) is
    built in-tree, binds to the ctypes library's cprrtc_plan, and declines
    (returns None) arguments it does not take instead of calling."""
    from paper_2505_06791_b200 import planner
    f = planner._fast()
    assert f is not None and f.__name__.endswith("_cprrtc_fast")
    z = np.zeros(7)
    assert f.plan_one(0, 0, z, z, 0, 0, 0, 0, 7) is None                   # NULL context: no call
    assert f.plan_one(1, 1, np.zeros(14)[::2], z, 0, 1, 1, 1, 7) is None    # strided start
    assert f.plan_one(1, 1, z.astype(np.float32), z, 0, 1, 1, 1, 7) is None
    with pytest.raises(TypeError):
        f.plan_one(0, 0, z)
