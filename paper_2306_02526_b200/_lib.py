"""ctypes binding of the C ABI declared in include/hpstep_b200.h.

The shared library is built in-tree (``paper_2306_02526_b200/lib``) by
``__graft_entry__.build()``.  There is no fallback: if the library or a CUDA
device is missing, every device entry point raises.
"""

import ctypes
import os

import numpy as np

from .errors import HpstepError, SingularMatrixError

_HERE = os.path.dirname(os.path.abspath(__file__))
# HPSB_LIB: an alternative build of the same library (A/B timing of two builds)
LIB_PATH = os.environ.get("HPSB_LIB") or os.path.join(_HERE, "lib", "libhpstep_b200.so")

HPS_OK = 0
HPS_PHASE_UP, HPS_PHASE_TOP, HPS_PHASE_DOWN, HPS_PHASE_ALL = 1, 2, 4, 7
HPS_ERR_SINGULAR = -3

c_int_p = ctypes.POINTER(ctypes.c_int)
c_ll_p = ctypes.POINTER(ctypes.c_longlong)
c_double_p = ctypes.POINTER(ctypes.c_double)


class PlanDesc(ctypes.Structure):
    _fields_ = [
        ("n1", ctypes.c_int), ("n2", ctypes.c_int), ("p", ctypes.c_int),
        ("depth", ctypes.c_int), ("N", ctypes.c_longlong),
        ("L", ctypes.c_int), ("ni", ctypes.c_int), ("nb", ctypes.c_int), ("nbd", ctypes.c_int),
        ("lvl_shape", c_int_p),
        ("lvl_i1a", ctypes.POINTER(c_int_p)), ("lvl_i3a", ctypes.POINTER(c_int_p)),
        ("lvl_i2b", ctypes.POINTER(c_int_p)), ("lvl_i3b", ctypes.POINTER(c_int_p)),
        ("lvl_gidx_bnd", ctypes.POINTER(c_int_p)), ("lvl_j3", ctypes.POINTER(c_int_p)),
        ("lvl_node_index", ctypes.POINTER(c_ll_p)),
        ("leaf_bnd_gidx", c_int_p), ("leaf_node_index", c_ll_p), ("boundary_ids", c_int_p),
        ("nparts", ctypes.c_int),
    ]


class BuildDesc(ctypes.Structure):
    _fields_ = [
        ("sigma", ctypes.c_double), ("dt_gamma", ctypes.c_double),
        ("shared_leaf", ctypes.c_int), ("keep_dtn", ctypes.c_int),
        ("coef", c_double_p), ("has_c1", ctypes.c_int), ("has_c2", ctypes.c_int),
        ("has_c", ctypes.c_int),
        ("D2x", c_double_p), ("D2y", c_double_p), ("D1x", c_double_p), ("D1y", c_double_p),
        ("D_bnd", c_double_p),
        ("layout", ctypes.c_int),
    ]


LAYOUT_PER_NODE = 0
LAYOUT_SHARED = 1


class DiscDesc(ctypes.Structure):
    _fields_ = [
        ("d1x", c_double_p), ("d2x", c_double_p), ("d1y", c_double_p), ("d2y", c_double_p),
        ("ex1", c_double_p), ("ex2", c_double_p), ("ey1", c_double_p), ("ey2", c_double_p),
        ("Lc", ctypes.c_int), ("coef", c_double_p),
        ("has_c1", ctypes.c_int), ("has_c2", ctypes.c_int), ("has_c", ctypes.c_int),
        ("leaf_bnd_sign", ctypes.POINTER(ctypes.c_byte)),
    ]


_vp = ctypes.c_void_p
_ll = ctypes.c_longlong
_i = ctypes.c_int

# exported symbols and their signatures (every name declared in include/hpstep_b200.h)
SIGNATURES = {
    "hps_version": (ctypes.c_int, []),
    "hps_launch_count": (ctypes.c_longlong, []),
    "hps_ops_level_pairs": (_i, [_vp]),
    "hps_last_error": (ctypes.c_char_p, []),
    "hps_last_error_node": (ctypes.c_longlong, []),
    "hps_plan_create": (ctypes.c_int, [ctypes.POINTER(PlanDesc), ctypes.POINTER(ctypes.c_void_p)]),
    "hps_plan_destroy": (None, [ctypes.c_void_p]),
    "hps_ops_build": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(BuildDesc), ctypes.c_void_p,
                                     ctypes.POINTER(ctypes.c_void_p)]),
    "hps_ops_destroy": (None, [ctypes.c_void_p]),
    "hps_ktimer_enable": (None, [_i]),
    "hps_plan_fused_level": (_i, [_vp]),
    "hps_workspace_level": (_i, [_vp, _i, _i, c_ll_p, c_ll_p]),
    "hps_top_level": (_i, [_vp, _i, _i, _i, _i, _i, _vp, _ll, _vp, _vp, ctypes.c_size_t, _vp]),
    "hps_ktimer_collect": (_i, [ctypes.c_char_p, _i, c_double_p, c_ll_p, _i]),
    "hps_merge_node": (_i, [_i, _vp, _i, _i, _i, _vp, _vp, _vp, _vp, _ll, _vp, _vp, _vp, _vp, _vp]),
    "hps_ops_device_bytes": (ctypes.c_size_t, [ctypes.c_void_p]),
    "hps_ops_get_leaf": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, c_double_p]),
    "hps_ops_get_merge": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                         c_double_p]),
    "hps_ops_set_leaf_fd": (ctypes.c_int, [ctypes.c_void_p, c_double_p, ctypes.c_int]),
    "hps_ops_dump_size": (ctypes.c_longlong, [ctypes.c_void_p]),
    "hps_ops_dump": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_longlong]),
    "hps_ops_load": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_longlong,
                                    ctypes.POINTER(ctypes.c_void_p)]),
    "hps_solve_workspace_bytes": (ctypes.c_size_t, [ctypes.c_void_p, ctypes.c_int]),
    "hps_solve": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_longlong,
                                 ctypes.c_void_p, ctypes.c_longlong, ctypes.c_void_p,
                                 ctypes.c_longlong, ctypes.c_double, ctypes.c_void_p,
                                 ctypes.c_longlong, ctypes.c_void_p, ctypes.c_size_t,
                                 ctypes.c_void_p]),
    "hps_solve_phase": (_i, [_vp, _i, _i, _i, _i, _vp, _ll, _vp, _ll, _vp, _ll, ctypes.c_double,
                             _vp, _ll, _vp, ctypes.c_size_t, _vp]),
    "hps_plan_partition": (_i, [_vp, _i, c_int_p, c_int_p, c_int_p, c_ll_p]),
    "hps_solve_stage": (_i, [_vp, _i, _vp, _ll, _vp, _ll, _vp, _ll, _vp, _ll, _vp, _vp, _vp, ctypes.c_size_t,
                             _vp]),
    "hps_solve_stage_terms": (_i, [_vp, _vp, _i, _vp, ctypes.POINTER(_vp), _vp, _vp, _vp, _vp, _vp, _vp,
                                   ctypes.c_size_t, _vp]),
    "hps_solve_stage_terms_k": (_i, [_vp, _i, _vp, _ll, _i, _vp, ctypes.POINTER(_vp), ctypes.POINTER(_ll), _vp, _ll,
                                     _vp, _ll, _vp, _ll, _vp, _vp, ctypes.c_size_t, _vp]),
    "hps_root_dirichlet_scratch": (ctypes.c_size_t, [_vp, _i]),
    "hps_root_dirichlet": (_i, [_vp, _i, _vp, _ll, _vp, _ll, _vp, ctypes.c_size_t, _vp]),
    "hps_leaf_lu": (_i, [_vp, _i, _i, _i, _vp, _ll, _vp, _ll, _vp, _vp]),
    "hps_disc_create": (_i, [_vp, ctypes.POINTER(DiscDesc), ctypes.POINTER(_vp)]),
    "hps_disc_destroy": (None, [_vp]),
    "hps_leaf_eval": (_i, [_vp, _i, _vp, _ll, _vp, _vp, _vp, _vp, _vp, _ll, _vp, _vp]),
    "hps_leaf_eval_range": (_i, [_vp, _i, _i, _i, _vp, _ll, _vp, _vp, _vp, _vp, _vp, _ll, _vp, _vp]),
    "hps_combine": (_i, [_i, _ll, _i, c_double_p, ctypes.POINTER(_vp), c_ll_p, _vp, _ll, _vp,
                         _vp]),
    "hps_combine_dev": (_i, [_i, _ll, _i, _vp, ctypes.POINTER(_vp), c_ll_p, _vp, _ll, _vp, _vp]),
    "hps_combine_dev_rows": (_i, [_i, _ll, _i, _vp, _ll, ctypes.POINTER(_vp), c_ll_p, _vp, _ll, _vp, _vp]),
    "hps_maxabs": (_i, [_i, _ll, _vp, _ll, _vp, _vp]),
    "hps_combine_bnd": (_i, [_vp, _i, _i, c_double_p, _vp, ctypes.POINTER(_vp), c_ll_p, _vp, _ll, _vp, _ll, _vp,
                             _vp]),
    "hps_put_boundary": (_i, [_vp, _i, _vp, _ll, _vp, _ll, _vp]),
}

_lib = None


def load():
    """Load the library (no CUDA device needed just to load it)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise HpstepError(
                f"CUDA library not built: {LIB_PATH} is missing "
                "(run `python -c 'import __graft_entry__ as g; g.build()'`)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def last_error():
    lib = load()
    return lib.hps_last_error().decode(errors="replace")


def check(rc, what):
    if rc == HPS_OK:
        return
    lib = load()
    msg = last_error()
    if rc == HPS_ERR_SINGULAR:
        # message ends with "[leaf node i]" / "[merge node i]" (SingularMatrixError context)
        body, _, ctx = msg.rpartition(" [")
        raise SingularMatrixError(body, context=ctx.rstrip("]") or None)
    raise HpstepError(f"{what} failed ({rc}): {msg} (node {lib.hps_last_error_node()})")


def int_ptr(a):
    return a.ctypes.data_as(c_int_p)


def ll_ptr(a):
    return a.ctypes.data_as(c_ll_p)


def dbl_ptr(a):
    return a.ctypes.data_as(c_double_p)


def as_i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def kernel_times(max_kernels=64):
    """{kernel name: (total ms, launches)} of the launches timed since
    hps_ktimer_enable(1) (hps_ktimer_collect; synchronises the device)."""
    import subprocess
    lib = load()
    names = ctypes.create_string_buffer(1 << 16)
    ms = (ctypes.c_double * max_kernels)()
    cnt = (ctypes.c_longlong * max_kernels)()
    n = lib.hps_ktimer_collect(names, len(names), ms, cnt, max_kernels)
    if n < 0:
        check(n, "hps_ktimer_collect")
    raw = names.value.decode().split("\n")[:n]
    try:
        dem = subprocess.run(["c++filt"], input="\n".join(raw), capture_output=True, text=True,
                             timeout=10).stdout.split("\n")[:n]
    except (OSError, subprocess.SubprocessError):
        dem = raw
    out = {}
    for i, name in enumerate(dem if len(dem) == n else raw):
        name = name.replace("hpsb::", "").replace("(anonymous namespace)::", "")
        name = name.split("(")[0].replace("void ", "").strip()
        a, c = out.get(name, (0.0, 0))
        out[name] = (a + ms[i], c + cnt[i])
    return out

