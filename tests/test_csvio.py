"""The reference's CSV formats (proj/src/csv.cpp) written from this library's results
(paper_1510_08982_b200/csvio.py), compared byte for byte with the reference's own output on
the same inputs (tests/golden/csv, made by tests/golden/gen_csv_golden.py)."""
import ctypes
import ctypes.util
import os

import numpy as np
import pytest

from helpers import SplitMix64

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "csv")


@pytest.fixture(scope="module")
def H():
    from paper_1510_08982_b200 import heat
    return heat


@pytest.fixture(scope="module")
def CSV():
    from paper_1510_08982_b200 import csvio
    return csvio


def _gold(name):
    with open(os.path.join(GOLD, name), "rb") as f:
        return f.read()


def _bytes(path):
    with open(path, "rb") as f:
        return f.read()


def test_format_double_matches_libc(CSV):
    # csv.cpp:11-15 is snprintf("%.17g"); glibc's own formatting is the oracle
    libc = ctypes.CDLL(ctypes.util.find_library("c"))
    buf = ctypes.create_string_buffer(64)
    gen = SplitMix64(1510)
    vals = [0.0, -0.0, 1.0, -1.0, 0.1, 1e300, -1e-300, 5e-324, 2.2250738585072014e-308,
            1.7976931348623157e308, 123456789012345680.0, 0.5, 1e16, 1e17, 9.999999999999999e22]
    for _ in range(3000):
        x = gen.next()
        v = np.frombuffer(np.uint64(x).tobytes(), np.float64)[0]
        if np.isfinite(v):
            vals.append(float(v))
        vals.append((gen.next_double() - 0.5) * 10.0 ** (gen.next_bounded(40) - 20))
    for v in vals:
        libc.snprintf(buf, 64, b"%.17g", ctypes.c_double(v))
        assert CSV.format_double(v) == buf.value.decode(), v


def _traj(H, steps, snaps, p, bc):
    return H.Trajectory([H.TemperatureField(s) for s in snaps], steps, p, bc)


def test_trajectory_csv_sync_golden(H, CSV, port, tmp_path):
    p = H.SolverParams.from_r(0.3)
    u0 = port.cosine_init(13)
    steps, snaps = port.sync_run(u0, p.r(), 0, 1.0, 0.0, 25, 5, record=True)
    out = str(tmp_path / "t.csv")
    CSV.emit_trajectory_csv(_traj(H, steps, snaps, p, H.BoundaryCondition.dirichlet(1, 0)), out)
    assert _bytes(out) == _gold("traj_sync.csv")


def test_trajectory_csv_async_golden_and_read_back(H, CSV, port, tmp_path):
    p = H.SolverParams.from_r(0.45)
    u0 = port.cosine_init(24)
    steps, snaps = port.async_run(u0, p.r(), 1, 0.0, 0.0, 8, 0, 3, seed=77, k_end=40, stride=7,
                                  record=True)
    out = str(tmp_path / "t.csv")
    CSV.emit_trajectory_csv(_traj(H, steps, snaps, p, H.BoundaryCondition.periodic()), out)
    assert _bytes(out) == _gold("traj_async.csv")
    back = CSV.read_trajectory_csv(out)  # %.17g round-trips bit-exactly (csv.hpp:11-12)
    assert back.steps == steps
    for j, s in enumerate(back.snapshots):
        assert np.array_equal(np.array(s).view(np.uint64), snaps[j].view(np.uint64))


def test_read_trajectory_csv_errors(CSV, tmp_path):
    bad = tmp_path / "bad.csv"
    bad.write_bytes(b"k,i,v\n")
    with pytest.raises(CSV.IoError, match="header"):
        CSV.read_trajectory_csv(str(bad))
    bad.write_bytes(b"k,i,u\n0,0,1\n0,2,1\n")
    with pytest.raises(CSV.IoError, match="non-contiguous"):
        CSV.read_trajectory_csv(str(bad))
    bad.write_bytes(b"k,i,u\n0,x,1\n")
    with pytest.raises(CSV.IoError, match="bad trajectory CSV row"):
        CSV.read_trajectory_csv(str(bad))
    with pytest.raises(CSV.IoError, match="cannot open"):
        CSV.read_trajectory_csv(str(tmp_path / "missing.csv"))


def test_bench_csv_golden(H, CSV, tmp_path):
    rows = [H.BenchRow(1000, H.ExecMode.Barriered, 5, 123456, 120000),
            H.BenchRow(1000, H.ExecMode.BarrierFree, 5, 9876, 9000)]
    out = str(tmp_path / "b.csv")
    CSV.emit_bench_csv(rows, out)
    assert _bytes(out) == _gold("bench.csv")


@pytest.mark.gpu
def test_ensemble_csv_golden(H, CSV, gpu, port, tmp_path):
    # the GPU ensemble (K6) written in the reference's format equals the
    # reference's own files for the same members
    cfg = H.EnsembleConfig(H.TemperatureField(port.cosine_init(16)), H.SolverParams.from_r(0.4),
                           H.BoundaryCondition.dirichlet(1.0, 0.0), H.PartitionSpec(16, 4),
                           H.DelayModel.uniform(2, 0), k_end=30, stride=10)
    res = H.ensemble_run(cfg, 3, 5)
    runs, stats = str(tmp_path / "r.csv"), str(tmp_path / "s.csv")
    CSV.emit_ensemble_csv(res, runs, stats)
    assert _bytes(runs) == _gold("ens_runs.csv")
    assert _bytes(stats) == _gold("ens_stats.csv")


@pytest.mark.gpu
def test_trajectory_csv_from_gpu_run(H, CSV, gpu, port, tmp_path):
    p = H.SolverParams.from_r(0.45)
    t = H.async_run(H.TemperatureField(port.cosine_init(24)), p, H.BoundaryCondition.periodic(),
                    H.PartitionSpec(24, 8), H.DelayModel.uniform(3, 77), 40, 7)
    out = str(tmp_path / "t.csv")
    CSV.emit_trajectory_csv(t, out)
    assert _bytes(out) == _gold("traj_async.csv")
