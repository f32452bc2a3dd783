"""Light-cone parity checks at full size.  TEST INFRASTRUCTURE ONLY.

SURVEY.md §8c "parity at scale": after k steps a point depends only on the
points at most k away (the asynchronous scheme reads neighbours one position
away too, at steps k - d), so a window of the initial field of half-width
k + 1 around a point determines it.  ``WindowCheck`` downloads such windows
from a device field BEFORE a run, and after the run compares every exact
point of each window (more than k points from a held window end, or up to a
true domain end) with the oracle's window run (``heat_oracle.c``
``orc_sync_window`` / ``orc_async_window``), bit for bit.  Used by
``tests/test_gpu_bench_parity.py`` and by bench.py's parity leg (the checker
of the timed run, never the thing timed).
"""
from __future__ import annotations

import concurrent.futures as cf
import os

import numpy as np


class WindowCheck:
    def __init__(self, n: int, k: int, centres, margin: int = 32):
        self.n, self.k = n, k
        self.windows = []  # (lo, w, a, b): exact points are lo + [a, b)
        for c in sorted(set(int(c) for c in centres)):
            lo = max(0, c - k - 1 - margin)
            hi = min(n, c + k + 2 + margin)
            a = 0 if lo == 0 else k + 1
            b = (hi - lo) if hi == n else (hi - lo) - k - 1
            if b > a:
                self.windows.append((lo, hi - lo, a, b))
        self.initial = None

    def capture(self, download_range) -> None:
        """download_range(offset, count) -> np.ndarray of the field BEFORE the run."""
        self.initial = [np.array(download_range(lo, w), dtype=np.float64)
                        for lo, w, _, _ in self.windows]

    def points(self) -> int:
        return sum(b - a for _, _, a, b in self.windows)

    def verify(self, download_range, advance) -> dict:
        """advance(window, lo) -> the window after the run (oracle); the run's
        result is read with download_range.  Returns {"ok", "points", "bad"}."""
        assert self.initial is not None, "capture() before the run"
        got = [np.array(download_range(lo + a, b - a), dtype=np.float64)
               for lo, _, a, b in self.windows]

        def one(i):
            lo, w, a, b = self.windows[i]
            exp = advance(self.initial[i], lo)[a:b]
            diff = np.nonzero(exp.view(np.uint64) != got[i].view(np.uint64))[0]
            return [(lo + a + int(j), float(got[i][j]), float(exp[j])) for j in diff[:4]]

        threads = max(1, min(len(self.windows), os.cpu_count() or 1))
        with cf.ThreadPoolExecutor(threads) as ex:  # ctypes releases the GIL
            bad = [x for r in ex.map(one, range(len(self.windows))) for x in r]
        return {"ok": not bad, "points": self.points(), "windows": len(self.windows),
                "bad": bad[:8]}
