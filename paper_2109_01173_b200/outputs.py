"""Trajectory outputs: the files the reference's DIB runner
writes (cli.py:106-139 via harness.py:424-491) — ``metrics.csv``, 16-bit PGM
frames of the snapshots and final states — with the frame normalisation and
quantisation done on the GPU (``sfb_frame_pgm16``): a full-size frame never
crosses PCIe as fp64.

Same bytes as the reference: RFC-4180 CSV with CRLF line endings and
shortest round-trip floats; binary 16-bit PGM, min-max normalised per frame,
constant frames as zeros.
"""

from __future__ import annotations

import csv
import os

import numpy as np

from . import _native as nat


def fmt(value) -> str:
    """Shortest round-trip text for floats; plain str otherwise (harness.py:424-430)."""
    if isinstance(value, (float, np.floating)):
        return repr(float(value))
    if isinstance(value, (int, np.integer)):
        return str(int(value))
    return str(value)


def write_csv(path, header, rows) -> None:
    """harness.py:433-440."""
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(header)
        for row in rows:
            w.writerow([fmt(v) for v in row])


def pgm_pixels(array):
    """Big-endian uint16 pixels of a frame (device normalisation); -> (numpy
    bytes-ready array, (min, max))."""
    t = nat.torch()
    A = nat.to_device(array)
    rows, cols = A.shape
    out = t.empty((rows, cols), dtype=t.int16, device="cuda")
    lohi = np.zeros(2)
    nat.check(nat.lib().sfb_frame_pgm16(nat.ptr(A), A.stride(0), rows, cols, out.data_ptr(), nat.dptr(lohi),
                                        nat.stream()), "pgm frame")
    return nat.to_host(out).view(">u2"), (float(lohi[0]), float(lohi[1]))


def write_pgm(path, array) -> None:
    """Binary 16-bit PGM, min-max normalised per frame (harness.py:475-491)."""
    px, _ = pgm_pixels(array)
    with open(path, "wb") as fh:
        fh.write(f"P5\n{px.shape[1]} {px.shape[0]}\n65535\n".encode())
        fh.write(px.tobytes())


def write_dib_outputs(out_dir, traj, tau: float) -> None:
    """metrics.csv, eta_<step>.pgm per snapshot, eta_final.pgm and
    theta_final.pgm of a two-species trajectory (cli.py:106-119)."""
    os.makedirs(out_dir, exist_ok=True)
    rows = [(k + 1, (k + 1) * tau, traj.increments[k, 0], traj.increments[k, 1], traj.iterations[k, 0],
             traj.iterations[k, 1]) for k in range(len(traj.times))]
    write_csv(os.path.join(out_dir, "metrics.csv"),
              ["step", "time", "increment_u", "increment_v", "pcg_iters_u", "pcg_iters_v"], rows)
    for step, eta, _theta in traj.snapshots:
        write_pgm(os.path.join(out_dir, f"eta_{step:06d}.pgm"), eta)
    write_pgm(os.path.join(out_dir, "eta_final.pgm"), traj.final[0])
    write_pgm(os.path.join(out_dir, "theta_final.pgm"), traj.final[1])
