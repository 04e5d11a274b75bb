"""Golden files of the reference's trajectory writers (harness.write_pgm,
harness.write_csv; harness.py:424-491), produced by running the UNMODIFIED
reference in this build container on seeded frames:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_outputs_golden.py

writes tests/golden/outputs.npz (inputs and the exact file bytes)."""

from __future__ import annotations

import os
import sys
import tempfile

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
sys.dont_write_bytecode = True

from sylfem.harness import write_csv, write_pgm  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "outputs.npz")


def frames():
    rng = np.random.default_rng(11)
    yield "random", rng.standard_normal((37, 53))
    ties = (rng.integers(0, 65535, 256) + 0.5) / 65535.0  # half-way pixel values (round half to even)
    ties[0], ties[1] = 0.0, 1.0
    yield "ties", ties.reshape(16, 16)
    yield "flat", np.full((9, 7), 0.5)
    yield "near_flat", 0.5 + 1e-15 * rng.standard_normal((9, 7))
    yield "dib_like", 1e-3 * rng.random((64, 48)) + 0.5


def main():
    g = {}
    with tempfile.TemporaryDirectory() as d:
        for name, a in frames():
            path = os.path.join(d, name + ".pgm")
            write_pgm(path, a)
            g[f"pgm/{name}/in"] = a
            g[f"pgm/{name}/bytes"] = np.frombuffer(open(path, "rb").read(), dtype=np.uint8)
        rng = np.random.default_rng(12)
        inc = rng.random((5, 2)) * 1e-3
        its = rng.integers(1, 50, (5, 2))
        rows = [(k + 1, (k + 1) * 1.25e-5, inc[k, 0], inc[k, 1], its[k, 0], its[k, 1]) for k in range(5)]
        path = os.path.join(d, "metrics.csv")
        write_csv(path, ["step", "time", "increment_u", "increment_v", "pcg_iters_u", "pcg_iters_v"], rows)
        g["csv/inc"], g["csv/its"] = inc, its
        g["csv/bytes"] = np.frombuffer(open(path, "rb").read(), dtype=np.uint8)
    np.savez_compressed(OUT, **g)
    print("wrote", OUT, len(g), "arrays")


if __name__ == "__main__":
    main()
