"""Persistence interop with the unmodified reference (stmesh, LM history CSV) and the model
bundle round trip (CPU)."""

import os

import numpy as np
import pytest

from paper_2305_15661_b200 import io as sio
from paper_2305_15661_b200.mesh import build_box_mesh, build_sector_mesh


def _ref():
    from oracle import strom_ref

    try:
        return strom_ref.load()
    except ImportError:
        pytest.skip("reference not installed")


def test_stmesh_round_trip_with_reference(tmp_path):
    S = _ref()
    for mesh, _ in (build_box_mesh(((0.0, 0.0), (2.0, 1.0)), 4, 3), build_sector_mesh(3, 5)):
        p1, p2 = os.path.join(tmp_path, "ours.stmesh"), os.path.join(tmp_path, "ref.stmesh")
        sio.save_mesh(mesh, p1)
        rm = S["meshing"].load_mesh(p1)  # the reference reads ours
        S["meshing"].save_mesh(rm, p2)
        assert open(p1).read() == open(p2).read()  # and writes the same bytes back
        back = sio.load_mesh(p2)
        for f in ("nodes", "elements", "interior_faces", "boundary_faces"):
            assert np.array_equal(getattr(back, f), getattr(mesh, f))
        assert back.boundary_tags == mesh.boundary_tags


def test_history_csv_matches_reference(tmp_path):
    S = _ref()
    h = np.array([[0, 1.5, 0.1, 0.2, 1e-4, 0.5], [1, 1.2, 0.01, 0.02, 5e-5, np.nan]])
    p1, p2 = os.path.join(tmp_path, "a.csv"), os.path.join(tmp_path, "b.csv")
    sio.history_csv(h, p1)
    S["lm"].history_csv(h, p2)
    assert open(p1).read() == open(p2).read()


def test_model_bundle_round_trip(tmp_path):
    from paper_2305_15661_b200.eqp import WeightVector
    from paper_2305_15661_b200.reduced import ReducedBases

    mesh, maps = build_box_mesh(((0.0, 0.0), (1.0, 1.0)), 2, 2, degree_sol=1)
    rng = np.random.default_rng(0)
    bases = ReducedBases(rng.standard_normal((maps.n_global_state, 2)), rng.standard_normal((maps.n_global_coord, 1)),
                         mesh.nodes.ravel())
    w = WeightVector(rng.uniform(0, 1, mesh.num_elements))
    snaps = [(rng.standard_normal(maps.n_global_state), mesh.nodes.ravel() + 1e-3)]
    p = os.path.join(tmp_path, "model.npz")
    sio.save_model(p, mesh, bases, w, [3, 1], snaps)
    m2, b2, w2, sel, sn = sio.load_model(p)
    assert np.array_equal(m2.elements, mesh.elements) and m2.boundary_tags == mesh.boundary_tags
    assert np.array_equal(b2.phi, bases.phi) and np.array_equal(w2.rho, w.rho) and sel == [3, 1]
    assert np.array_equal(sn[0][0], snaps[0][0])
    mp = os.path.join(tmp_path, "metrics.csv")
    sio.greedy_metrics_csv([{"j": 1, "mu": [6.0, 0.0475], "T_rho": 0.5, "active": 3}], mp)
    lines = open(mp).read().splitlines()
    assert lines[0].startswith("j,mu,") and lines[1].startswith("1,6.0 0.0475,")
