"""The reference's CSV emitters and reader (proj/include/heat/csv.hpp, src/csv.cpp) for the
results of the GPU path: trajectories, ensembles, bench rows.

Every float is rendered as C's ``%.17g`` (csv.cpp:11-15). Python's ``%`` formatting and glibc's
``snprintf`` both round the exact binary value correctly to 17 significant digits, so the bytes
match; ``tests/test_csvio.py`` checks this against libc's own ``snprintf``. Files are written in
binary mode with LF endings (csv.cpp:19-23).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .heat import BenchRow, EnsembleResult, Trajectory, to_string


class IoError(RuntimeError):
    """config.hpp IoError: a file could not be opened, written or parsed."""


def format_double(v: float) -> str:
    """csv.cpp:11-15"""
    return "%.17g" % v


def _open(path: str):
    try:
        return open(path, "wb")
    except OSError as exc:
        raise IoError("cannot open for writing: " + path) from exc


def emit_trajectory_csv(traj: Trajectory, path: str) -> None:
    """csv.cpp:32-42: header "k,i,u", one row per recorded (step, grid point)."""
    with _open(path) as out:
        out.write(b"k,i,u\n")
        for s, snap in enumerate(traj.snapshots):
            v = snap.values() if hasattr(snap, "values") else np.asarray(snap, np.float64)
            k = traj.steps[s]
            out.write("".join(f"{k},{i},{'%.17g' % x}\n" for i, x in enumerate(v.tolist())).encode())


@dataclass
class TrajectoryData:
    """csv.hpp:22-25"""

    steps: list = field(default_factory=list)
    snapshots: list = field(default_factory=list)


def read_trajectory_csv(path: str) -> TrajectoryData:
    """csv.cpp:44-68: rows grouped by step; point indices must be contiguous."""
    try:
        f = open(path, "rb")
    except OSError as exc:
        raise IoError("cannot open for reading: " + path) from exc
    data = TrajectoryData()
    with f:
        lines = f.read().decode().split("\n")
    if not lines or lines[0] != "k,i,u":
        raise IoError("bad trajectory CSV header in " + path)
    for line in lines[1:]:
        if not line:
            continue
        parts = line.split(",")
        try:
            if len(parts) != 3:
                raise ValueError
            k, i, u = int(parts[0]), int(parts[1]), float(parts[2])
        except ValueError:
            raise IoError("bad trajectory CSV row in " + path + ": " + line) from None
        if not data.steps or data.steps[-1] != k:
            data.steps.append(k)
            data.snapshots.append([])
        if i != len(data.snapshots[-1]):
            raise IoError("non-contiguous point index in " + path)
        data.snapshots[-1].append(u)
    return data


def emit_ensemble_csv(res: EnsembleResult, runs_path: str, stats_path: str) -> None:
    """csv.cpp:70-88: "k,run,norm2" per (run, step), then "k,mean,std" per step."""
    with _open(runs_path) as out:
        out.write(b"k,run,norm2\n")
        for j, series in enumerate(res.norm_series):
            out.write("".join(f"{k},{j},{'%.17g' % series[s]}\n"
                              for s, k in enumerate(res.steps)).encode())
    with _open(stats_path) as out:
        out.write(b"k,mean,std\n")
        out.write("".join(f"{k},{'%.17g' % res.mean_series[s]},{'%.17g' % res.std_series[s]}\n"
                          for s, k in enumerate(res.steps)).encode())


def emit_bench_csv(rows: list[BenchRow], path: str) -> None:
    """csv.cpp:90-97: "N,mode,reps,median_ns,min_ns"."""
    with _open(path) as out:
        out.write(b"N,mode,reps,median_ns,min_ns\n")
        out.write("".join(f"{r.n_points},{to_string(r.mode)},{r.reps},{r.median_ns},{r.min_ns}\n"
                          for r in rows).encode())
