"""ctypes binding of the C ABI declared in include/strom_b200.h."""

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.environ.get("STROM_SO") or os.path.join(HERE, "_strom_b200.so")

OBJECTIVE, DERIVS, CONTRIB, CONTRIB_SPLIT, RESIDUAL, RESNORM2, CONTRIB_LPROWS, ELEMJAC, ELEMJAC_ENRICHED = range(9)


class MeshDesc(C.Structure):
    _fields_ = [("num_elements", C.c_int32), ("num_nodes", C.c_int32), ("elem_nodes", C.c_void_p),
                ("nodes", C.c_void_p), ("nbr_elem", C.c_void_p), ("face_info", C.c_void_p)]


class LawDesc(C.Structure):
    _fields_ = [("law_id", C.c_int32), ("n_comp", C.c_int32), ("n_mu", C.c_int32), ("params", C.c_double * 8)]


class QuadDesc(C.Structure):
    _fields_ = [("p", C.c_int32), ("nb", C.c_int32), ("nq", C.c_int32), ("ns", C.c_int32), ("nf", C.c_int32),
                ("phi", C.c_void_p), ("dphi", C.c_void_p), ("wq", C.c_void_p), ("bary", C.c_void_p),
                ("trace", C.c_void_p), ("ws", C.c_void_p), ("s", C.c_void_p), ("fnodes", C.c_void_p)]


class DistDesc(C.Structure):
    _fields_ = [("kappa", C.c_double), ("eps", C.c_double)]


EXPORTS = ("strom_create", "strom_set_bases", "strom_set_offsets", "strom_set_test_space", "strom_reserve", "strom_eval", "strom_eval_host",
           "strom_degenerate_elements",
           "strom_lm_solve", "strom_lm_stats", "strom_lm_timing", "strom_lm_rows", "strom_profile", "strom_profile_ms", "strom_last_error", "strom_destroy")

_lib = None


class ExtensionMissing(RuntimeError):
    pass


def load(path=SO_PATH):
    """Load the CUDA library; fails loudly — there is no CPU fallback."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ExtensionMissing(f"{path} not built; run `python -m paper_2305_15661_b200.build`")
    lib = C.CDLL(path)
    vp, i32 = C.c_void_p, C.c_int32
    lib.strom_create.argtypes = [C.POINTER(MeshDesc), C.POINTER(LawDesc), C.POINTER(QuadDesc),
                                 C.POINTER(DistDesc), C.c_int, C.POINTER(vp)]
    lib.strom_set_bases.argtypes = [vp, vp, i32, vp, i32, vp, vp]
    lib.strom_reserve.argtypes = [vp, i32, i32]
    lib.strom_set_test_space.argtypes = [vp, i32, vp, vp, vp]
    lib.strom_set_offsets.argtypes = [vp, vp, C.c_int64, vp, C.c_int64]
    lib.strom_eval.argtypes = [vp, i32, vp, vp, vp, i32, vp, vp, i32, vp, vp, vp, i32]
    lib.strom_eval_host.argtypes = [vp, i32, vp, vp, vp, i32, vp, vp, i32, vp, C.c_int64, vp, vp]
    lib.strom_degenerate_elements.argtypes = [vp, i32, vp, i32]
    lib.strom_lm_solve.argtypes = [vp, vp, vp, vp, i32, vp, vp, i32, vp, vp, vp, vp]
    lib.strom_lm_stats.argtypes = [vp, vp]
    lib.strom_lm_timing.argtypes = [vp, vp]
    lib.strom_lm_rows.argtypes = [vp, vp]
    lib.strom_profile.argtypes = [vp, i32]
    lib.strom_profile_ms.argtypes = [vp, C.POINTER(i32)]
    lib.strom_profile_ms.restype = C.c_double
    lib.strom_last_error.restype = C.c_char_p
    lib.strom_destroy.argtypes = [vp]
    lib.strom_destroy.restype = None
    _lib = lib
    return lib


def check(rc, what="strom call"):
    if rc < 0:
        msg = load().strom_last_error().decode()
        raise RuntimeError(f"{what} failed ({rc}): {msg}")
    return rc
