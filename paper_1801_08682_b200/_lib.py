"""ctypes binding of ``include/aderdg_b200.h`` (the C ABI of the CUDA library).

The library is built in-tree (``paper_1801_08682_b200/libaderdg_b200.so``) by
``build.py``.  There is no CPU fallback: a missing library or a failing CUDA
call raises ``DeviceError``.
"""

import ctypes
import os

import numpy as np

from .errors import (ConfigurationError, DeviceError, NumericalError,
                     PredictorFailureError)

LIB_NAME = "libaderdg_b200.so"
LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), LIB_NAME)
# the same sources built with ADG_DEBUG_CHECKS (build.py): record stamps, bounds,
# poisoned shared memory, jittered barriers, reversed cell order
DEBUG_LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libaderdg_b200_debug.so")
_debug_lib = None

ADG_OK, ADG_ERR_CONFIG, ADG_ERR_NUMERICAL, ADG_ERR_RUNTIME, ADG_ERR_PREDICTOR = 0, 2, 3, 4, 5
ADG_BUF_Q, ADG_BUF_D, ADG_BUF_TRACE0, ADG_BUF_TRACE1, ADG_BUF_REDUCE = range(5)
ADG_PART_ALL, ADG_PART_INTERIOR, ADG_PART_BOUNDARY = range(3)
ADG_TIMED_KERNEL_EVENTS = 1   # adg_run_timed_ex flags

#: every symbol the header declares (checked by tests/test_abi.py)
EXPORTS = (
    "adg_create", "adg_destroy", "adg_set_operators", "adg_set_stream",
    "adg_load_state", "adg_store_state", "adg_seed", "adg_step", "adg_run",
    "adg_step_records",
    "adg_sync", "adg_step_count", "adg_rerun_count", "adg_sweep_count",
    "adg_time_control", "adg_picard_histogram", "adg_error_info",
    "adg_last_error", "adg_layout_info", "adg_buffer", "adg_phase_seed",
    "adg_phase_seed_finish", "adg_phase_rerun", "adg_phase_sweep",
    "adg_phase_finish", "adg_trace_parity", "adg_flush_l2", "adg_reset", "adg_set_dt_new",
    "adg_run_timed", "adg_run_timed_ex", "adg_phase_sweep_part", "adg_set_limiter", "adg_troubled_flags",
    "adg_step_host", "adg_nccl_unique_id", "adg_nccl_init", "adg_run_timed_mgpu", "adg_run_timed_mgpu_ex",
    "adg_group_init", "adg_group_seed", "adg_group_run", "adg_set_option", "adg_device_count",
)

ADG_OPT_GRAPH, ADG_OPT_COND_RERUN, ADG_OPT_HOST_CHUNKS, ADG_OPT_FUSE_FINISH, ADG_OPT_PERSISTENT = 1, 2, 3, 4, 5


class AdgConfig(ctypes.Structure):
    _fields_ = [
        ("d", ctypes.c_int), ("p", ctypes.c_int), ("L", ctypes.c_int),
        ("cfl", ctypes.c_double), ("c_dt", ctypes.c_double),
        ("creeping", ctypes.c_int), ("forced_dt", ctypes.c_double),
        ("inject_rerun", ctypes.c_int), ("spike_step", ctypes.c_int),
        ("spike_factor", ctypes.c_double), ("device", ctypes.c_int),
        ("rank", ctypes.c_int), ("world", ctypes.c_int), ("halo_mode", ctypes.c_int),
        ("driver_mode", ctypes.c_int), ("system", ctypes.c_int),
        ("velocity", ctypes.c_double * 3), ("boundary", ctypes.c_int),
    ]


class AdgStepRecord(ctypes.Structure):
    _fields_ = [
        ("step", ctypes.c_int), ("reruns", ctypes.c_int),
        ("T", ctypes.c_double), ("dt_old", ctypes.c_double),
        ("dt_new", ctypes.c_double), ("dt_adm", ctypes.c_double),
        ("picard_iters", ctypes.c_longlong), ("predicts", ctypes.c_longlong),
        ("troubled", ctypes.c_longlong),
    ]


class AdgLayout(ctypes.Structure):
    _fields_ = [
        ("n_cells_global", ctypes.c_int), ("n_cells_local", ctypes.c_int),
        ("cell_offset", ctypes.c_int), ("planes_local", ctypes.c_int),
        ("plane_cells", ctypes.c_int), ("record_doubles", ctypes.c_int),
        ("faces_per_cell", ctypes.c_int), ("state_doubles", ctypes.c_size_t),
    ]


_lib = None


def _preload_nccl():
    """The library resolves NCCL with dlopen("libnccl.so.2") when a multi-GPU path
    first needs it; make that the torch-bundled NCCL (the one torch.distributed
    uses) even in processes that never import torch.  Absent: the system library."""
    try:
        import nvidia.nccl
        base = list(nvidia.nccl.__path__)[0]
        ctypes.CDLL(os.path.join(base, "lib", "libnccl.so.2"), mode=ctypes.RTLD_GLOBAL)
    except (ImportError, OSError, IndexError):
        pass


def load_library(path=None, debug=False):
    """Load (once) and prototype the CUDA library; raise if it is missing."""
    global _lib, _debug_lib
    if debug:
        if _debug_lib is None:
            _debug_lib = load_library(DEBUG_LIB_PATH)
        return _debug_lib
    if _lib is not None and path is None:
        return _lib
    p = path or LIB_PATH
    if not os.path.exists(p):
        raise DeviceError(f"native library {p} is missing: run `python -c 'import "
                          f"__graft_entry__ as g; g.build()'` (there is no CPU fallback)")
    _preload_nccl()
    lib = ctypes.CDLL(p)
    H = ctypes.c_void_p
    dp = ctypes.POINTER(ctypes.c_double)
    proto = {
        "adg_create": (ctypes.c_int, [ctypes.POINTER(AdgConfig), ctypes.POINTER(H)]),
        "adg_destroy": (None, [H]),
        "adg_set_operators": (ctypes.c_int, [H, dp, dp, dp, dp, dp, dp]),
        "adg_set_stream": (ctypes.c_int, [H, ctypes.c_void_p]),
        "adg_load_state": (ctypes.c_int, [H, dp, ctypes.c_size_t]),
        "adg_store_state": (ctypes.c_int, [H, dp, ctypes.c_size_t]),
        "adg_seed": (ctypes.c_int, [H]),
        "adg_step": (ctypes.c_int, [H, ctypes.POINTER(AdgStepRecord)]),
        "adg_run": (ctypes.c_int, [H, ctypes.c_int, ctypes.POINTER(AdgStepRecord)]),
        "adg_step_records": (ctypes.c_int, [H, ctypes.c_int, ctypes.c_int,
                                            ctypes.POINTER(AdgStepRecord)]),
        "adg_sync": (ctypes.c_int, [H]),
        "adg_step_count": (ctypes.c_int, [H]),
        "adg_rerun_count": (ctypes.c_int, [H]),
        "adg_sweep_count": (ctypes.c_int, [H]),
        "adg_time_control": (ctypes.c_int, [H, dp, dp, dp, dp]),
        "adg_picard_histogram": (ctypes.c_int, [H, ctypes.POINTER(ctypes.c_longlong), ctypes.c_int]),
        "adg_error_info": (ctypes.c_int, [H, ctypes.POINTER(ctypes.c_int),
                                          ctypes.POINTER(ctypes.c_longlong),
                                          ctypes.POINTER(ctypes.c_int), dp]),
        "adg_last_error": (ctypes.c_char_p, [H]),
        "adg_layout_info": (ctypes.c_int, [H, ctypes.POINTER(AdgLayout)]),
        "adg_buffer": (ctypes.c_int, [H, ctypes.c_int, ctypes.POINTER(ctypes.c_void_p),
                                      ctypes.POINTER(ctypes.c_size_t)]),
        "adg_phase_seed": (ctypes.c_int, [H]),
        "adg_phase_seed_finish": (ctypes.c_int, [H]),
        "adg_phase_rerun": (ctypes.c_int, [H]),
        "adg_phase_sweep": (ctypes.c_int, [H]),
        "adg_phase_sweep_part": (ctypes.c_int, [H, ctypes.c_int]),
        "adg_set_limiter": (ctypes.c_int, [H, dp, dp, ctypes.POINTER(ctypes.c_int),
                                           ctypes.POINTER(ctypes.c_int),
                                           ctypes.POINTER(ctypes.c_longlong), ctypes.c_double]),
        "adg_troubled_flags": (ctypes.c_int, [H, ctypes.POINTER(ctypes.c_ubyte), ctypes.c_size_t]),
        "adg_step_host": (ctypes.c_int, [H, dp, dp, ctypes.POINTER(AdgStepRecord)]),
        "adg_phase_finish": (ctypes.c_int, [H]),
        "adg_trace_parity": (ctypes.c_int, [H]),
        "adg_flush_l2": (ctypes.c_int, [H]),
        "adg_reset": (ctypes.c_int, [H]),
        "adg_set_dt_new": (ctypes.c_int, [H, ctypes.c_double]),
        "adg_run_timed": (ctypes.c_int, [H, ctypes.c_int, dp]),
        "adg_run_timed_ex": (ctypes.c_int, [H, ctypes.c_int, ctypes.c_int, dp]),
        "adg_nccl_unique_id": (ctypes.c_int, [ctypes.POINTER(ctypes.c_ubyte)]),
        "adg_nccl_init": (ctypes.c_int, [H, ctypes.POINTER(ctypes.c_ubyte), ctypes.c_int, ctypes.c_int]),
        "adg_run_timed_mgpu": (ctypes.c_int, [H, ctypes.c_int, dp]),
        "adg_run_timed_mgpu_ex": (ctypes.c_int, [H, ctypes.c_int, ctypes.c_int, dp]),
        "adg_group_init": (ctypes.c_int, [ctypes.POINTER(H), ctypes.c_int]),
        "adg_group_seed": (ctypes.c_int, [ctypes.POINTER(H), ctypes.c_int]),
        "adg_group_run": (ctypes.c_int, [ctypes.POINTER(H), ctypes.c_int, ctypes.c_int,
                                         ctypes.POINTER(AdgStepRecord)]),
        "adg_set_option": (ctypes.c_int, [H, ctypes.c_int, ctypes.c_int]),
        "adg_device_count": (ctypes.c_int, []),
    }
    for name, (res, args) in proto.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _lib = lib
    return lib


def dptr(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


class Handle:
    """Owning wrapper of one ``adg_handle``; maps status codes to exceptions."""

    def __init__(self, cfg, debug=False):
        self.lib = load_library(debug=debug)
        self.h = ctypes.c_void_p()
        st = self.lib.adg_create(ctypes.byref(cfg), ctypes.byref(self.h))
        self.check(st, "adg_create")

    def close(self):
        if self.h:
            self.lib.adg_destroy(self.h)
            self.h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def last_error(self):
        msg = self.lib.adg_last_error(self.h)
        return msg.decode() if msg else ""

    def error_info(self):
        kind, cell, step, val = ctypes.c_int(), ctypes.c_longlong(), ctypes.c_int(), ctypes.c_double()
        self.lib.adg_error_info(self.h, ctypes.byref(kind), ctypes.byref(cell), ctypes.byref(step),
                                ctypes.byref(val))
        return kind.value, cell.value, step.value, val.value

    def check(self, status, what):
        if status == ADG_OK:
            return
        msg = self.last_error() if self.h else ""
        if status == ADG_ERR_CONFIG:
            raise ConfigurationError(msg or what)
        if status == ADG_ERR_NUMERICAL:
            _, cell, step, _ = self.error_info()
            raise NumericalError(msg, cell_index=cell, step=step)
        if status == ADG_ERR_PREDICTOR:
            _, cell, _, _ = self.error_info()
            raise PredictorFailureError(cell)
        raise DeviceError(f"{what}: {msg}")

    def call(self, name, *args):
        st = getattr(self.lib, name)(self.h, *args)
        self.check(st, name)

    def layout(self):
        lay = AdgLayout()
        self.call("adg_layout_info", ctypes.byref(lay))
        return lay

    def buffer(self, which):
        ptr, nbytes = ctypes.c_void_p(), ctypes.c_size_t()
        self.call("adg_buffer", which, ctypes.byref(ptr), ctypes.byref(nbytes))
        return ptr.value, nbytes.value

    def time_control(self):
        v = [ctypes.c_double() for _ in range(4)]
        self.call("adg_time_control", *[ctypes.byref(x) for x in v])
        return tuple(x.value for x in v)

    def step_records(self, first, count):
        recs = (AdgStepRecord * max(count, 1))()
        self.call("adg_step_records", int(first), int(count), recs)
        return list(recs)[:count]

    def picard_histogram(self, bins=32):
        arr = (ctypes.c_longlong * bins)()
        self.call("adg_picard_histogram", arr, bins)
        return np.array(arr[:], dtype=np.int64)


class DeviceArray:
    """Minimal ``__cuda_array_interface__`` view of a handle-owned buffer so that
    torch (NCCL plumbing) can address it without copies."""

    def __init__(self, ptr, shape, typestr, device):
        self.__cuda_array_interface__ = {
            "shape": tuple(shape), "typestr": typestr, "data": (ptr, False),
            "version": 3, "strides": None,
        }
        self.device = device
