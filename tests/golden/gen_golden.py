"""Generate tests/golden/golden.json from the REFERENCE itself.

Run in the build container, where /root/reference exists and
oracle/_ref/libheat_ref.so can be compiled from it (oracle/Makefile):

    python tests/golden/gen_golden.py

Every value below is produced by the reference's own code (heat::sync_run,
heat::async_run, heat::exec_run, heat::sample_delay, heat::cosine_init,
SolverParams::checked) through oracle/ref_shim.cpp.  The fixtures travel with
the repo so the GPU box (no /root/reference) and the CPU tests can check the
oracle port and the CUDA path against them.
"""
from __future__ import annotations

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

from helpers import SplitMix64, fnv1a64, random_divisor, random_field  # noqa: E402
from oracle import oracle as O  # noqa: E402


def hexs(v):
    return [float(x).hex() for x in v]


def main():
    R = O.ref()
    P = O.port()
    out = {"source": "reference (oracle/_ref/libheat_ref.so built from /root/reference/proj/src)"}

    # --- delay streams (test_async_sim.cpp:55-98) -----------------------------
    out["delay_streams"] = [
        {"law": 0, "q": 4, "d": 0, "p": 0.5, "seed": 42, "k": 100, "count": 8,
         "values": R.delay_stream(0, 4, 0, 0.5, 42, 100, 8)},
        {"law": 1, "q": 4, "d": 2, "p": 0.5, "seed": 77, "k": 100, "count": 4,
         "values": R.delay_stream(1, 4, 2, 0.5, 77, 100, 4)},
        {"law": 2, "q": 6, "d": 0, "p": 0.7, "seed": 99, "k": 1000, "count": 64,
         "values": R.delay_stream(2, 6, 0, 0.7, 99, 1000, 64)},
        {"law": 0, "q": 8, "d": 0, "p": 0.5, "seed": 1234, "k": 3, "count": 32,
         "values": R.delay_stream(0, 8, 0, 0.5, 1234, 3, 32)},
    ]
    # --- parameters -----------------------------------------------------------
    out["r_bits"] = {"checked(0.5,0.01,0.1)": R.checked_r(0.5, 0.01, 0.1).hex(),
                     "0.25": (0.25).hex(), "0.4": (0.4).hex()}
    # --- cosine IC (core.cpp:29-39) ------------------------------------------
    out["cosine_init_100_fnv"] = fnv1a64(R.cosine_init(100))

    # --- BASELINE configs 1 and 2 (sine IC) -------------------------------------
    u = P.prepare_initial(P.sine_init(1024), O.DIRICHLET, 0.0, 0.0)
    out["sine_1024_fnv"] = fnv1a64(u)
    fin = R.sync_run(u, 0.25, O.DIRICHLET, 0.0, 0.0, 1000)
    out["cfg1"] = {"fnv": fnv1a64(fin), "u512": fin[512].hex(), "l2": P.l2_norm(fin).hex()}
    out["cfg2"] = []
    for seed in (1, 42):
        for q in (2, 3):
            fin = R.async_run(u, 0.25, O.DIRICHLET, 0.0, 0.0, 128, O.UNIFORM, q, seed=seed,
                              k_end=1000)
            out["cfg2"].append({"seed": seed, "q": q, "fnv": fnv1a64(fin)})

    # --- small random cases with full inputs (acceptance.cpp:67-99 style) -----
    cases = []
    gen = SplitMix64(20261018)
    for t in range(40):
        n = 3 + gen.next_bounded(40)
        r = 0.5 * (gen.next_double() * 0.999 + 0.001)
        periodic = int(gen.next() & 1)
        u0 = random_field(gen, n)
        c1, c2 = (0.0, 0.0) if periodic else (float(u0[0]), float(u0[-1]))
        k = 1 + gen.next_bounded(200)
        per = random_divisor(gen, n)
        q = 1 + gen.next_bounded(6)
        law = int(gen.next_bounded(2))
        fd = int(gen.next_bounded(q - 1)) if law == 1 else 0
        gp = 0.1 + 0.8 * gen.next_double() if law == 2 else 0.5
        seed = gen.next()
        sync = R.sync_run(u0, r, periodic, c1, c2, k)
        asy = R.async_run(u0, r, periodic, c1, c2, per, law, q, fd, gp, seed, k)
        cases.append({"n": n, "r": r.hex(), "bc": periodic, "c1": c1.hex(), "c2": c2.hex(),
                      "k": k, "u0": hexs(u0), "per_pe": per, "q": q, "law": law, "d": fd,
                      "p": gp.hex(), "seed": seed, "sync_final": hexs(sync),
                      "async_final": hexs(asy)})
    out["cases"] = cases

    # --- ensembles (analysis.cpp:51-104) --------------------------------------
    r_paper = R.checked_r(0.5, 0.01, 0.1)
    cos100 = R.cosine_init(100)
    ens = []
    for (bc, c1, c2, per, law, q, fd, k, stride, runs, base) in (
            (O.DIRICHLET, 1.0, 0.0, 1, O.UNIFORM, 5, 0, 3000, 1000, 4, 1000),
            (O.PERIODIC, 0.0, 0.0, 10, O.FIXED, 4, 2, 2500, 700, 3, 7),
            (O.PERIODIC, 0.0, 0.0, 1, O.UNIFORM, 3, 0, 2000, 0, 2, 42)):
        steps, norms, terms, mean, std, spread = R.ensemble_run(
            cos100, r_paper, bc, c1, c2, per, law, q, fd, k, stride, runs, base)
        ens.append({"bc": bc, "c1": c1, "c2": c2, "per_pe": per, "law": law, "q": q, "d": fd,
                    "k": k, "stride": stride, "runs": runs, "base": base, "steps": steps,
                    "norms": [hexs(row) for row in norms],
                    "terminal_fnv": [fnv1a64(t) for t in terms],
                    "mean": hexs(mean), "std": hexs(std)})
    out["ensembles"] = ens
    # acceptance.cpp criteria 2-3 (M=50, N=100, one point per PE, q=5, 2e5 steps)
    crit = {}
    for name, bc, c1, c2 in (("dirichlet", O.DIRICHLET, 1.0, 0.0), ("periodic", O.PERIODIC, 0.0, 0.0)):
        steps, norms, terms, mean, std, spread = R.ensemble_run(
            cos100, r_paper, bc, c1, c2, 1, O.UNIFORM, 5, 0, 200000, 200000, 50, 1000)
        crit[name] = {"terminal_fnv": [fnv1a64(t) for t in terms],
                      "spread_mean_temp": float(spread[0]).hex(),
                      "spread_norm": float(spread[1]).hex(), "mean": hexs(mean)}
    out["acceptance_ensembles"] = crit

    # --- KATs of test_sync.cpp ------------------------------------------------
    out["kat_sync_step_dirichlet"] = hexs(R.sync_step([1.0, 0.0, 0.0], 0.5, O.DIRICHLET, 1.0, 0.0))
    out["kat_sync_step_periodic"] = hexs(R.sync_step([2.0, 0.0, 1.0], 0.25, O.PERIODIC))

    path = os.path.join(HERE, "golden.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", path)


if __name__ == "__main__":
    main()
