"""Algorithm 1 orchestration on the GPU (greedy.greedy_train) with synthetic HDM snapshots:
seed, greedy searches over the candidate set, Gram-Schmidt basis growth, weight retraining
(the reference's train_weights with the GPU operator swapped in when the reference is
installed), exhaustion error."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


def test_greedy_train_bookkeeping():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2305_15661_b200 import configs, laws as L
    from paper_2305_15661_b200.eqp import WeightVector
    from paper_2305_15661_b200.greedy import CandidateSetExhausted, greedy_train, seed_index
    from paper_2305_15661_b200.lm import LmConfig

    case = configs.sector_rom_case(n_radial=3, n_circ=6, ku=2, kx=1, frac_active=0.5, rho_scale=2.0, P=1, seed=95,
                                   wall="extrapolate")
    geom, ne = case.geom, case.mesh.num_elements
    cands = np.array([[2.0], [2.5], [3.0], [3.5], [4.0]])
    rng = np.random.default_rng(1)
    bump = 1.0 + 0.02 * rng.standard_normal(ne * 24)

    def hdm_snapshot(mu, x):  # synthetic "HDM" state: freestream(mu) with a fixed perturbation
        return np.tile(L.euler_freestream(float(mu[0])), ne * 6) * bump, x

    def train(bases, guess, mus):  # all-ones weights keep the bookkeeping test independent of the LP
        return WeightVector.ones(ne)

    try:  # the reference's EQP LP with the GPU operator swapped in
        from oracle import strom_ref

        S = strom_ref.load()
        from paper_2305_15661_b200 import dropin

        def train(bases, guess, mus):  # noqa: F811
            undo = dropin.install(lm=True)
            try:
                cfg = S["eqp"].EqpTrainingConfig(delta=0.5, xi=np.asarray(mus))
                rb = S["reduced"].ReducedBases(bases.phi, bases.psi, bases.ref_coords)
                return S["eqp"].train_weights(case.law, case.mesh, case.maps, rb, guess, cfg, case.dist,
                                              S["lm"].LmConfig(max_iters=5))
            finally:
                undo()
    except ImportError:
        pass

    st = greedy_train(case.law, geom, cands, hdm_snapshot, 3, case.dist, train, LmConfig(max_iters=5))
    assert st.selected[0] == seed_index(cands) == 2
    assert len(set(st.selected)) == 3 and st.bases.phi.shape[1] == 3 and st.bases.psi.shape[1] == 3
    assert np.allclose(st.bases.phi.T @ st.bases.phi, np.eye(3), atol=1e-12)
    assert np.allclose(st.bases.psi.T @ st.bases.psi, np.eye(3), atol=1e-12)
    assert [m["j"] for m in st.metrics] == [1, 2, 3] and all(np.all(st.weights.rho >= 0.0) for _ in [0])
    with pytest.raises(CandidateSetExhausted):
        greedy_train(case.law, geom, cands[:2], hdm_snapshot, 3, case.dist, train, LmConfig(max_iters=3))
