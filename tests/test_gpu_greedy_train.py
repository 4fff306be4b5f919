"""Algorithm 1 orchestration on the GPU (greedy.greedy_train) with synthetic HDM snapshots on
the reference's Burgers space-time law: seed at the candidate centroid (SPEC example: the
middle of the 3 x 3 grid on [3, 9] x [0.02, 0.075]), greedy searches over the candidate set,
Gram-Schmidt basis growth, weight retraining (the reference's train_weights with the GPU
operator swapped in when the reference is installed), exhaustion error."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


def test_greedy_train_bookkeeping():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2305_15661_b200 import configs, laws as L
    from paper_2305_15661_b200.eqp import WeightVector
    from paper_2305_15661_b200.greedy import CandidateSetExhausted, greedy_train
    from paper_2305_15661_b200.lm import LmConfig
    from paper_2305_15661_b200.mesh import build_box_mesh, get_geometry

    mesh, maps = build_box_mesh(((0.0, 0.0), (2.0, 1.0)), 4, 3, degree_sol=2, n_comp=1)
    law = L.burgers_spacetime()
    geom, ne = get_geometry(mesh, maps), mesh.num_elements
    cands = np.array([[a, b] for a in (3.0, 6.0, 9.0) for b in (0.02, 0.0475, 0.075)])
    xy = np.repeat(mesh.nodes[mesh.elements[:, :3]].mean(axis=1), 6, axis=0)  # element centroids per DG node

    nodes = mesh.nodes

    def hdm_snapshot(mu, x):  # synthetic "HDM" state and an aligned mesh: mu-dependent smooth fields
        d = 1e-3 * np.stack([np.sin(mu[0] * nodes[:, 1]), np.cos(40.0 * mu[1] * nodes[:, 0])], 1)
        return 1.0 + 0.1 * np.sin(mu[0] * xy[:, 0] + 40.0 * mu[1] * xy[:, 1]), x + d.ravel()

    train = lambda bases, guess, mus: WeightVector.ones(ne)  # noqa: E731  (LP-independent bookkeeping)
    try:  # the reference's EQP LP with the GPU operator swapped in
        from oracle import strom_ref
        from paper_2305_15661_b200 import dropin

        S = strom_ref.load()

        def train(bases, guess, mus):  # noqa: F811
            undo = dropin.install(lm=True)
            try:
                cfg = S["eqp"].EqpTrainingConfig(delta=0.5, xi=np.asarray(mus))
                rb = S["reduced"].ReducedBases(bases.phi, bases.psi, bases.ref_coords)
                rmesh, rmaps = S["meshing"].build_structured_mesh(((0.0, 0.0), (2.0, 1.0)), 4, 3, degree_sol=2, n_comp=1)
                sguess = S["eqp"].WeightVector(np.asarray(guess.rho))
                return S["eqp"].train_weights(S["conslaw"].burgers_spacetime(), rmesh, rmaps, rb, sguess, cfg,
                                              S["distortion"].DistortionConfig(1e-3), S["lm"].LmConfig(max_iters=5))
            finally:
                undo()
    except ImportError:
        pass

    dist = configs.DistortionConfig(1e-3)
    st = greedy_train(law, geom, cands, hdm_snapshot, 3, dist, train, LmConfig(max_iters=5))
    assert np.allclose(cands[st.selected[0]], [6.0, 0.0475])  # seed: the centroid of the grid
    assert len(set(st.selected)) == 3 and st.bases.phi.shape[1] == 3 and st.bases.psi.shape[1] == 3
    assert np.allclose(st.bases.phi.T @ st.bases.phi, np.eye(3), atol=1e-12)
    assert np.allclose(st.bases.psi.T @ st.bases.psi, np.eye(3), atol=1e-12)
    assert [m["j"] for m in st.metrics] == [1, 2, 3] and np.all(np.asarray(st.weights.rho) >= 0.0)
    assert all(m["psi_grown"] for m in st.metrics[1:])
    with pytest.raises(CandidateSetExhausted):
        greedy_train(law, geom, cands[:2], hdm_snapshot, 3, dist, train, LmConfig(max_iters=3))


def test_greedy_train_with_fullspace_callbacks():
    """Algorithm 1 end to end on the GPU with the built-in full-space callbacks: HDM solves
    (fullspace.solve_hdm) + full-space tracking for the snapshots, the alignment problem of
    Eq. align0 (tracking.TrackingProblem with the current state basis) before each of them."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import warnings

    from paper_2305_15661_b200 import configs, laws as L
    from paper_2305_15661_b200.eqp import WeightVector
    from paper_2305_15661_b200.fullspace import assemble_global
    from paper_2305_15661_b200.greedy import greedy_train, tracking_alignment, tracking_snapshot
    from paper_2305_15661_b200.lm import LmConfig
    from paper_2305_15661_b200.mesh import build_box_mesh, get_geometry

    mesh, maps = build_box_mesh(((0.0, 0.0), (1.0, 1.0)), 3, 3, degree_sol=2, n_comp=4)
    law = L.euler(tags={"left": "freestream", "bottom": "freestream", "right": "extrapolate", "top": "extrapolate"})
    geom, ne = get_geometry(mesh, maps, 6), mesh.num_elements
    dist = configs.DistortionConfig(1e-3)
    cands = np.array([[2.0], [2.5], [3.0], [3.5]])
    train = lambda bases, guess, mus: WeightVector.ones(ne)  # noqa: E731
    snap = tracking_snapshot(law, geom, dist, LmConfig(max_iters=3))
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")  # uniform flow: the aligned mesh is X, Psi is not grown
        st = greedy_train(law, geom, cands, snap, 2, dist, train, LmConfig(max_iters=4),
                          align=tracking_alignment(law, geom, dist, LmConfig(max_iters=3)))
    assert st.j == 2 and st.bases.phi.shape[1] == 2 and len(set(st.selected)) == 2
    X = mesh.nodes.ravel()
    for (U, x), i in zip(st.snapshots, st.selected):
        # the snapshots solve the DG system on their meshes, and boundary nodes stay on the box
        R = assemble_global(law, mesh, maps, U, x, cands[i], want_jacobians=False, geom=geom)[0]
        assert np.linalg.norm(R) < 1e-8
        assert np.allclose(U.reshape(-1, 4), L.euler_freestream(cands[i][0]), atol=1e-7)  # uniform freestream
        d = (x - X).reshape(-1, 2)
        on_v = (np.abs(mesh.nodes[:, 0]) < 1e-12) | (np.abs(mesh.nodes[:, 0] - 1.0) < 1e-12)
        on_h = (np.abs(mesh.nodes[:, 1]) < 1e-12) | (np.abs(mesh.nodes[:, 1] - 1.0) < 1e-12)
        assert np.max(np.abs(d[on_v, 0]), initial=0.0) <= 1e-12 and np.max(np.abs(d[on_h, 1]), initial=0.0) <= 1e-12
