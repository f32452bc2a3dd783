"""CPU: the C-ABI library loads, exports every symbol include/heat_b200.h
declares, the ctypes table matches the header, and without a GPU every compute
entry point fails loudly (HEAT_ENODEV) instead of falling back to the CPU."""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_1510_08982_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "heat_b200.h")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(heat_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_entry_points():
    names = declared()
    for must in ("heat_sync_run", "heat_async_run", "heat_exec_run", "heat_sync_step",
                 "heat_sync_run_f32", "heat_plan_create", "heat_plan_sync_advance"):
        assert must in names


def test_library_exports_all_declared_symbols():
    lib = ctypes.CDLL(_lib.LIB_PATH, mode=os.RTLD_NOW)  # fails on unresolved symbols
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_ctypes_table_matches_header():
    assert set(declared()) == set(_lib.SIGNATURES)


def test_no_silent_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    from paper_1510_08982_b200 import heat as H
    with pytest.raises(H.NativeUnavailable):
        H.sync_run(H.cosine_init(10), H.SolverParams.from_r(0.5),
                   H.BoundaryCondition.dirichlet(1.0, 0.0), 5)
    with pytest.raises(H.NativeUnavailable):
        H.async_final(np.zeros(16), H.SolverParams.from_r(0.5), H.BoundaryCondition.periodic(),
                      H.PartitionSpec(16, 4), H.DelayModel.uniform(2, 1), 5)
    assert _lib.lib().heat_device_count() == 0


def test_host_side_helpers_without_gpu():
    L = _lib.lib()
    assert L.heat_trajectory_length(10, 10, 3) == 5      # steps 0,3,6,9,10
    assert L.heat_trajectory_length(2000, 250, 0) == 4    # default stride 100
    assert L.heat_slab_halo() == 64
    v, nb, out, sp = ctypes.c_int(), ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    assert L.heat_sync_kernel_info(ctypes.byref(v), ctypes.byref(nb), ctypes.byref(out),
                                   ctypes.byref(sp)) == 0
    assert v.value in (32, 48, 64) and nb.value in (1, 2) and sp.value in (32, 64)
    # a K1 tile (32V - 2H exact points) or a K1s chunk (a first tile, then
    # tiles of 32V - H exact points)
    tile, col = 32 * v.value - 2 * sp.value, 32 * v.value - sp.value
    assert out.value == tile or (out.value - tile) % col == 0
    L.heat_set_strict_finite_checks(1)
    assert L.heat_strict_finite_checks() == 1
    L.heat_set_strict_finite_checks(0)
    from paper_1510_08982_b200 import heat as H
    assert [H.sample_delay_at(H.DelayModel.uniform(4, 42), j, 100) for j in range(8)] == \
        [1, 3, 2, 0, 2, 2, 1, 0]


def test_python_mirror_validation():
    from paper_1510_08982_b200 import heat as H
    with pytest.raises(H.DomainError):
        H.SolverParams.checked(0.5, 1.0, 1.0 - 1e-9)  # r > 0.5
    assert H.SolverParams.checked(0.5, 0.01, 0.1).r().hex() == "0x1.ffffffffffffep-2"
    with pytest.raises(H.DomainError):
        H.TemperatureField([1.0, 2.0])
    with pytest.raises(H.DomainError):
        H.TemperatureField([1.0, float("nan"), 2.0])
    with pytest.raises(H.DomainError):
        H.PartitionSpec(100, 7)
    p = H.PartitionSpec(100, 25)
    assert p.pe_count() == 4 and p.crosses(24, 25) and not p.crosses(25, 26)
    lg = H.LagStats()
    lg.merge(H.LagStats(2, 0, 1, [1, 1], 0))
    assert lg.mean() == 0.5
