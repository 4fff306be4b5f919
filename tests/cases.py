"""Golden-vector cases shared by the oracle pin tests and the GPU parity tests.

Each golden ``.npz`` (tests/golden/make_golden.py, produced by the
unmodified reference) stores the seeded inputs; the mesh, law and rule are
rebuilt here from this package (the mesh builders reproduce the reference
mesher's connectivity exactly — tests/test_host.py checks it).
"""

import os

import numpy as np

from paper_2305_15661_b200 import configs, laws as L
from paper_2305_15661_b200.mesh import build_box_mesh

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    with np.load(os.path.join(GOLDEN, f"{name}.npz"), allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


def build(name):
    """(case, golden dict) with the case's arrays replaced by the stored inputs."""
    g = load(name)
    if name == "strip":
        case = configs.strip_case(ncell=16, n_active=10, P=3, seed=11, boundary_in_sample=False)
    elif name in ("euler_square_q6", "euler_square_default"):
        case = configs.euler_square_case(n=4, ku=16, kx=8, seed=12, quad_order=6 if name.endswith("q6") else None,
                                         per_component=False)
    elif name.startswith("tracking"):
        case = configs.euler_square_case(n=4, ku=16, kx=8, seed=61, quad_order=6 if name.endswith("q6") else None)
        case.law = L.euler(tags={"left": "freestream", "bottom": "freestream", "right": "extrapolate",
                                 "top": "extrapolate"})
    elif name == "sector":
        case = configs.sector_rom_case(n_radial=4, n_circ=6, ku=6, kx=4, frac_active=0.25, rho_scale=4.0, P=2, seed=13,
                                   wall="extrapolate")
    elif name == "degenerate":
        case = configs.euler_square_case(n=4, ku=4, kx=2, seed=14, quad_order=6, per_component=False)
    elif name.startswith("burgers_st") or name.startswith("linadv"):
        p = int(g["p"])
        box = g["box"]
        nx, ny = (int(v) for v in g["nxny"])
        mesh, maps = build_box_mesh(box, nx, ny, degree_sol=p, n_comp=1)
        if name.startswith("burgers_st"):
            law = L.burgers_spacetime()
        else:
            law = L.linear_advection((1.0, 0.5) if name.endswith("p2") else (-0.7, 1.0),
                                     manufactured=L.ExpManufactured() if name.startswith("linadv_ms") else None)
        case = configs.Case(name, law, mesh, maps, None, None, None, None, None, None, None)
    else:
        raise KeyError(name)
    case.phi, case.psi, case.ref_coords = g["phi"], g["psi"], g["ref_coords"]
    case.mus = g["mus"]
    case.rho = g["rho"] if g["rho"].size else None
    case.quad_order = None if int(g["quad_order"]) < 0 else int(g["quad_order"])
    case.state_offset = g.get("state_offset")
    case.kappa, case.eps = float(g["kappa"]), float(g["eps"])
    return case, g


EVAL_CASES = ["strip", "euler_square_q6", "euler_square_default", "sector", "burgers_st_p1", "burgers_st_p2",
              "linadv_p1", "linadv_p2", "linadv_ms_p1", "linadv_ms_p2"]


def rel_err(a, b, scale=None):
    a, b = np.asarray(a, dtype=float), np.asarray(b, dtype=float)
    s = np.max(np.abs(b)) if scale is None else scale
    return float(np.max(np.abs(a - b)) / max(s, 1e-300)) if a.size else 0.0
