"""ctypes binding of libmhdg.so (the C ABI declared in include/mhdg.h).

The shared library is built in-tree (``python -c "import __graft_entry__ as g;
g.build()"`` or ``make -C paper_2402_11361_b200/csrc``).  There is no fallback:
if the library or a CUDA device is missing, every device operation raises.
"""

from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# MHDG_LIB: an alternative build of the same library (A/B measurements of compile-time variants)
LIB_PATH = os.environ.get("MHDG_LIB") or os.path.join(HERE, "libmhdg.so")

MHDG_OK = 0
MHDG_ERR_ADMISSIBILITY = 1
MHDG_ERR_FACTORIZATION = 2
MHDG_ERR_PRECONDITIONER = 3
MHDG_ERR_CONFIG = 4
MHDG_ERR_CUDA = 5

_dp = C.c_void_p  # device pointer


class Disc(C.Structure):
    _fields_ = [
        ("dim", C.c_int), ("ns", C.c_int), ("nf", C.c_int),
        ("n_mac", C.c_int), ("n_faces", C.c_int), ("n_trace", C.c_int),
        ("L", C.c_int), ("Lf", C.c_int),
        ("n_sub", C.c_int), ("nloc", C.c_int), ("nq", C.c_int),
        ("n_tri", C.c_int), ("nlocf", C.c_int), ("nqf", C.c_int),
        ("face_fac", C.c_double),
        ("mass", _dp), ("mass_inv", _dp), ("minv_d", _dp), ("weak_deriv", _dp), ("gf", _dp), ("face_mass", _dp),
        ("face_vol_nodes", _dp), ("sub_conn", _dp), ("phi_vol", _dp), ("grad_ref", _dp), ("w_ref", _dp),
        ("tri_conn", _dp), ("phi_face", _dp), ("w_face_ref", _dp), ("pm_vol", _dp), ("pm_face", _dp),
        ("vn_ptr", _dp), ("vn_sub", _dp), ("vf_ptr", _dp), ("vf_ent", _dp), ("fn_ptr", _dp), ("fn_ent", _dp),
        ("det", _dp), ("inv_jac", _dp), ("normals", _dp), ("areas", _dp), ("h_sub", _dp),
        ("gather", _dp), ("scatter_src", _dp),
        ("bc_kind", _dp), ("wall_e", _dp), ("wall_u", _dp), ("u_dir", _dp), ("source", _dp),
        ("face_macros", _dp), ("face_locals", _dp),
        ("n_face_nodes", C.c_int), ("node_to_face", _dp), ("minv_d_face", _dp),
        ("n_grad_cls", C.c_int), ("grad_cls", _dp), ("grad_cls_of", _dp),
    ]


class Flow(C.Structure):
    _fields_ = [("gamma", C.c_double), ("prandtl", C.c_double), ("re_acoustic", C.c_double),
                ("mach_ref", C.c_double), ("mu", C.c_double), ("re_flow", C.c_double)]


class Stage(C.Structure):
    _fields_ = [("dt_coeff", C.c_double), ("hist", _dp), ("pseudo_dt", C.c_double), ("supg_dt", C.c_double)]


class Blocks(C.Structure):
    _fields_ = [("state_state", _dp), ("face_state_trace", _dp), ("face_trace_state", _dp),
                ("face_trace_trace", _dp), ("wdgdq_vol", _dp), ("wdgdq_face", _dp), ("trace_face_scale", _dp)]


class Frozen(C.Structure):
    _fields_ = [("supg_tau", _dp), ("supg_jac", _dp), ("face_stab", _dp), ("face_visc_state", _dp)]


class Factors(C.Structure):
    _fields_ = [("lu", _dp), ("perm", _dp), ("scratch", _dp), ("work", _dp), ("kind", C.c_int),
                ("scratch_macros", C.c_int)]


_lib = None


def lib():
    """Load libmhdg.so once; raise if it is not built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is not built; run __graft_entry__.build() (no CPU fallback exists)")
        L = C.CDLL(LIB_PATH)
        P = C.POINTER
        sigs = {
            "mhdg_assemble": [P(Disc), P(Flow), P(Stage), _dp, _dp, _dp, _dp, _dp, _dp, _dp, C.c_int, P(Blocks),
                              P(Frozen), P(Frozen), _dp, _dp],
            "mhdg_condense": [P(Disc), P(Blocks), P(Factors), _dp, _dp],
            "mhdg_schur_matrix": [P(Disc), P(Blocks), P(Factors), _dp],
            "mhdg_lu_factor": [P(Disc), P(Factors), _dp, _dp],
            "mhdg_lu_solve": [P(Disc), P(Factors), _dp, _dp, _dp],
            "mhdg_apply_trace": [P(Disc), P(Blocks), P(Factors), _dp, _dp, _dp, _dp],
            "mhdg_apply_trace_local": [P(Disc), P(Blocks), P(Factors), _dp, _dp, _dp],
            "mhdg_face_reduce": [P(Disc), _dp, _dp, _dp],
            "mhdg_condensed_rhs": [P(Disc), P(Blocks), P(Factors), _dp, _dp, _dp, _dp, _dp, _dp],
            "mhdg_recover": [P(Disc), P(Blocks), P(Factors), _dp, _dp, _dp, _dp, _dp, _dp],
            "mhdg_gradient_refresh": [P(Disc), _dp, _dp, _dp, _dp],
            "mhdg_precond_build": [P(Disc), P(Blocks), _dp, _dp, _dp],
            "mhdg_precond_apply": [P(Disc), _dp, _dp, _dp, _dp],
            "mhdg_precond_build_ext": [P(Disc), P(Blocks), _dp, _dp, _dp, _dp],
            "mhdg_side_blocks": [P(Disc), P(Blocks), _dp, _dp, C.c_int, _dp, _dp],
            "mhdg_ahat_form": [P(Disc), P(Blocks), P(Factors), _dp, _dp, _dp, _dp, _dp],
            "mhdg_ahat_apply": [P(Disc), _dp, _dp, _dp, _dp, _dp],
            "mhdg_ahat_apply_local": [P(Disc), _dp, _dp, _dp, _dp],
            "mhdg_apply_trace_local_range": [P(Disc), P(Blocks), P(Factors), _dp, _dp, C.c_int, C.c_int, _dp],
            "mhdg_halo_gather": [C.c_longlong, _dp, _dp, _dp, _dp],
            "mhdg_halo_scatter": [C.c_longlong, _dp, _dp, _dp, C.c_int, _dp],
            "mhdg_face_reduce_remote": [P(Disc), _dp, _dp, _dp, C.c_int, _dp, _dp],
            "mhdg_assemble_window": [P(Disc), P(Flow), P(Stage), _dp, _dp, _dp, _dp, _dp, _dp, C.c_int, P(Blocks),
                                     P(Frozen), C.c_int, C.c_int, _dp, _dp],
            "mhdg_condense_window": [P(Disc), P(Blocks), P(Factors), C.c_int, C.c_int, _dp, _dp],
            "mhdg_apply_trace_local_window": [P(Disc), P(Blocks), P(Factors), _dp, _dp, C.c_int, C.c_int, _dp],
            "mhdg_condensed_rhs_local_window": [P(Disc), P(Blocks), P(Factors), _dp, _dp, _dp, C.c_int, C.c_int, _dp],
            "mhdg_recover_window": [P(Disc), P(Blocks), P(Factors), _dp, _dp, _dp, _dp, _dp, C.c_int, C.c_int, _dp],
            "mhdg_face_sum_window": [P(Disc), P(Blocks), _dp, C.c_int, C.c_int, _dp],
            "mhdg_precond_build_sums": [P(Disc), _dp, _dp, _dp, _dp],
            "mhdg_face_reduce_axpy": [P(Disc), _dp, _dp, C.c_double, _dp, _dp],
        }
        for name, args in sigs.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = C.c_int
        L.mhdg_set_stream_enabled.argtypes = [C.c_int]
        L.mhdg_set_stream_enabled.restype = None
        L.mhdg_factor_max_n.argtypes = [C.c_int]
        L.mhdg_factor_max_n.restype = C.c_int
        L.mhdg_packed_lu_size.argtypes = [C.c_int]
        L.mhdg_packed_lu_size.restype = C.c_longlong
        L.mhdg_launch_count.argtypes = []
        L.mhdg_launch_count.restype = C.c_longlong
        L.mhdg_apply_work_size.argtypes = [P(Disc)]
        L.mhdg_apply_work_size.restype = C.c_longlong
        L.mhdg_set_apply_split.argtypes = [C.c_int]
        L.mhdg_set_apply_split.restype = None
        L.mhdg_set_stream_prefetch.argtypes = [C.c_int]
        L.mhdg_set_stream_prefetch.restype = None
        L.mhdg_set_lu_panel.argtypes = [C.c_int, C.c_int]
        L.mhdg_set_lu_panel.restype = None
        L.mhdg_set_lu_small.argtypes = [C.c_int]
        L.mhdg_set_lu_small.restype = None
        L.mhdg_set_lu_grid.argtypes = [C.c_int]
        L.mhdg_set_lu_grid.restype = None
        L.mhdg_set_lu_l2mode.argtypes = [C.c_int]
        L.mhdg_set_lu_l2mode.restype = None
        L.mhdg_set_precond_variant.argtypes = [C.c_int]
        L.mhdg_set_precond_variant.restype = None
        L.mhdg_set_couplings_kernel.argtypes = [C.c_int]
        L.mhdg_set_couplings_kernel.restype = None
        L.mhdg_set_schur_variant.argtypes = [C.c_int]
        L.mhdg_set_schur_variant.restype = None
        L.mhdg_icgs.argtypes = [C.c_int, C.c_int, _dp, C.c_longlong, _dp, _dp, _dp, _dp]
        L.mhdg_icgs.restype = C.c_int
        L.mhdg_vec_pass.argtypes = [C.c_longlong, C.c_int, _dp, C.c_longlong, _dp, _dp, C.c_int, _dp, _dp, _dp]
        L.mhdg_vec_pass.restype = C.c_int
        L.mhdg_icgs_scratch_size.argtypes = [C.c_int]
        L.mhdg_icgs_scratch_size.restype = C.c_longlong
        L.mhdg_timeline_begin.argtypes = [C.c_int]
        L.mhdg_timeline_begin.restype = C.c_int
        L.mhdg_timeline_end.argtypes = [C.POINTER(C.c_double), C.POINTER(C.c_int)]
        L.mhdg_timeline_end.restype = C.c_int
        _lib = L
    return _lib


# the drop-in C ABI (include/mhdg.h)
EXPORTED = (
    "mhdg_assemble", "mhdg_condense", "mhdg_schur_matrix", "mhdg_lu_factor", "mhdg_lu_solve",
    "mhdg_apply_trace", "mhdg_apply_trace_local", "mhdg_face_reduce", "mhdg_condensed_rhs", "mhdg_recover",
    "mhdg_gradient_refresh", "mhdg_precond_build", "mhdg_precond_apply", "mhdg_launch_count",
    "mhdg_packed_lu_size", "mhdg_precond_build_ext", "mhdg_side_blocks",
    "mhdg_apply_work_size", "mhdg_timeline_begin", "mhdg_timeline_end", "mhdg_icgs", "mhdg_icgs_scratch_size",
    "mhdg_ahat_form", "mhdg_ahat_apply", "mhdg_ahat_apply_local", "mhdg_factor_max_n",
    "mhdg_vec_pass", "mhdg_apply_trace_local_range", "mhdg_halo_gather", "mhdg_halo_scatter",
    "mhdg_face_reduce_remote", "mhdg_assemble_window", "mhdg_condense_window", "mhdg_apply_trace_local_window",
    "mhdg_condensed_rhs_local_window", "mhdg_recover_window", "mhdg_face_sum_window", "mhdg_precond_build_sums",
    "mhdg_face_reduce_axpy",
)
# diagnostic A/B knobs (csrc/mhdg_tuning.h; not part of the drop-in ABI)
TUNING = (
    "mhdg_set_schur_variant", "mhdg_set_lu_panel", "mhdg_set_lu_l2mode", "mhdg_set_lu_grid", "mhdg_set_lu_small", "mhdg_set_apply_split",
    "mhdg_set_stream_enabled", "mhdg_set_stream_prefetch", "mhdg_stream_grid", "mhdg_set_precond_variant",
    "mhdg_set_couplings_kernel",
)


TIMELINE_SLOTS = ("apply_pre", "apply_si", "apply_post", "apply_fused", "apply_generic", "face_reduce",
                  "schur", "factor", "pack", "assemble", "apply_ahat", "icgs", "precond_build", "precond_apply",
                  "halo")


class Timeline:
    """Per-kernel CUDA-event timeline of the library's launches (mhdg_timeline_*)."""

    def __init__(self, capacity: int = 4096):
        self.capacity = capacity
        self.ms, self.counts = {}, {}

    def __enter__(self):
        check(lib().mhdg_timeline_begin(self.capacity), "mhdg_timeline_begin")
        return self

    def __exit__(self, *exc):
        ms, cnt = (C.c_double * 16)(), (C.c_int * 16)()
        check(lib().mhdg_timeline_end(ms, cnt), "mhdg_timeline_end")
        for i, name in enumerate(TIMELINE_SLOTS):
            if cnt[i]:
                self.ms[name], self.counts[name] = ms[i], cnt[i]


def check(rc: int, what: str) -> None:
    if rc != MHDG_OK:
        raise RuntimeError(f"{what} failed with status {rc}")


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None -> NULL)."""
    return None if t is None else t.data_ptr()


def arg(t, numel: int | None = None, what: str = "argument"):
    """Validate a float64 device array handed to the C ABI and return it contiguous.

    The caller must keep the returned tensor alive until the library call has been
    issued (bind it to a local): a temporary from ``.contiguous()`` that is freed
    before the call can be handed straight back by the caching allocator to the
    next temporary, so two arguments would alias."""
    import torch

    if t.dtype != torch.float64:
        raise TypeError(f"{what}: expected float64, got {t.dtype}")
    if t.device.type != "cuda":
        raise ValueError(f"{what}: expected a CUDA tensor, got device {t.device}")
    if numel is not None and t.numel() != numel:
        raise ValueError(f"{what}: expected {numel} entries, got {t.numel()}")
    return t.contiguous()
