"""Trajectory outputs: the oracle restatement of the
reference writers against golden files the reference wrote (CPU), and the
product's device PGM quantisation / CSV writer byte for byte (GPU)."""

import os
import tempfile

import numpy as np
import pytest

import oracle as orc

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "outputs.npz"))
FRAMES = sorted({k.split("/")[1] for k in GOLD.files if k.startswith("pgm/")})
HEADER = ["step", "time", "increment_u", "increment_v", "pcg_iters_u", "pcg_iters_v"]


def csv_rows():
    inc, its = GOLD["csv/inc"], GOLD["csv/its"]
    return [(k + 1, (k + 1) * 1.25e-5, inc[k, 0], inc[k, 1], its[k, 0], its[k, 1]) for k in range(len(inc))]


@pytest.mark.parametrize("name", FRAMES)
def test_oracle_pgm_matches_reference_bytes(name):
    assert orc.pgm_bytes(GOLD[f"pgm/{name}/in"]) == GOLD[f"pgm/{name}/bytes"].tobytes()


def test_oracle_csv_matches_reference_bytes():
    assert orc.csv_text(HEADER, csv_rows()).encode() == GOLD["csv/bytes"].tobytes()


def test_product_csv_matches_reference_bytes():
    from paper_2109_01173_b200.outputs import write_csv
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "metrics.csv")
        write_csv(p, HEADER, csv_rows())
        assert open(p, "rb").read() == GOLD["csv/bytes"].tobytes()


@pytest.mark.gpu
@pytest.mark.parametrize("name", FRAMES)
def test_device_pgm_matches_reference_bytes(name):
    from paper_2109_01173_b200.outputs import write_pgm
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "f.pgm")
        write_pgm(p, GOLD[f"pgm/{name}/in"])
        assert open(p, "rb").read() == GOLD[f"pgm/{name}/bytes"].tobytes()


@pytest.mark.gpu
def test_dib_outputs_written():
    import paper_2109_01173_b200 as pb
    from paper_2109_01173_b200.outputs import write_dib_outputs
    p = pb.dib_presets("spots_worms").replace(rho=400.0)
    x, y = pb.build_direction_sets(pb.SQUARE, 1, 15, pb.BCKind.NEUMANN, lumped=True)
    e0, t0 = pb.initial_fields((y.q, x.q), pb.InitialData(amplitude=2e-3, seed=5))
    tau = 5e-3 / p.rho
    tr = pb.imex_euler_rds(pb.SQUARE, x, y, 1.0, p.d_theta, pb.dib_kinetics_pair(p), p.rho, (e0, t0),
                           pb.TimeGrid(tau, 4 * tau), lumped=True, snapshot_every=2)
    with tempfile.TemporaryDirectory() as d:
        write_dib_outputs(d, tr, tau)
        assert sorted(os.listdir(d)) == ["eta_000002.pgm", "eta_000004.pgm", "eta_final.pgm", "metrics.csv",
                                         "theta_final.pgm"]
        assert open(os.path.join(d, "eta_final.pgm"), "rb").read() == orc.pgm_bytes(tr.final[0])
        rows = [(k + 1, (k + 1) * tau, tr.increments[k, 0], tr.increments[k, 1], tr.iterations[k, 0],
                 tr.iterations[k, 1]) for k in range(4)]
        assert open(os.path.join(d, "metrics.csv")).read() == orc.csv_text(HEADER, rows).replace("\r\n", "\n")
