"""ctypes binding of liblevyh_b200.so (include/levyh_b200.h).

The native library is the only compute path: importing the package on a
machine without it raises, and every GPU operation raises when no CUDA device
is present.  There is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liblevyh_b200.so")

LH_OK, LH_EINVAL, LH_ESINGULAR, LH_ETYPE, LH_ECUDA, LH_ENOMEM, LH_ERANK, LH_EINTERNAL = range(8)


class HConfigC(C.Structure):
    _fields_ = [("n_min", C.c_int32), ("n_block", C.c_int32), ("eta", C.c_double),
                ("eps1", C.c_double), ("kcap", C.c_int32), ("max_aca_rank", C.c_int32),
                ("aca_tol", C.c_double)]


class MeasureC(C.Structure):
    _fields_ = [("kind", C.c_int32), ("c", C.c_double), ("s", C.c_double), ("C", C.c_double),
                ("G", C.c_double), ("M", C.c_double), ("Y", C.c_double),
                ("table_dev", C.c_void_p)]


class Cn2dEntriesC(C.Structure):
    _fields_ = [("nx", C.c_int32), ("which", C.c_int32), ("h", C.c_double), ("eps_sq", C.c_double),
                ("scale", C.c_double), ("a", C.c_double), ("b", C.c_double), ("c", C.c_double),
                ("lam", C.c_double), ("dt", C.c_double), ("order_dev", C.c_void_p)]


class CNParamsC(C.Structure):
    _fields_ = [("h", C.c_double), ("N", C.c_int64), ("M", C.c_int64), ("rho_r", C.c_double),
                ("tail", C.c_double), ("m2", C.c_double), ("a", C.c_double), ("b", C.c_double),
                ("c", C.c_double), ("dt", C.c_double)]


# (name, restype, argtypes) for every symbol declared in include/levyh_b200.h
P, I32, I64, D = C.c_void_p, C.c_int32, C.c_int64, C.c_double
SIGNATURES = [
    ("lh_ctx_create", C.c_int, [C.c_int, P, C.POINTER(P)]),
    ("lh_ctx_destroy", None, [P]),
    ("lh_ctx_last_error", C.c_char_p, [P]),
    ("lh_ctx_synchronize", C.c_int, [P]),
    ("lh_ctx_stream", C.c_void_p, [P]),
    ("lh_version", C.c_int, []),
    ("lh_tree_build", C.c_int, [P, P, I64, C.c_int, C.c_int, C.POINTER(P)]),
    ("lh_tree_destroy", None, [P]),
    ("lh_tree_num_nodes", I64, [P]),
    ("lh_tree_nodes", C.c_int, [P, P, P, P]),
    ("lh_tree_order", C.c_int, [P, P]),
    ("lh_partition", C.c_int, [P, P, C.c_int, C.c_int, D, P, P, P]),
    ("lh_plan_stats", C.c_int, [P, P, C.c_int, C.c_int, D, C.c_int, P]),
    ("lh_hmat_build_toeplitz", C.c_int, [P, P, P, P, C.POINTER(HConfigC), C.POINTER(P)]),
    ("lh_hmat_build_dense", C.c_int, [P, P, P, P, I64, C.c_int, C.POINTER(HConfigC), C.POINTER(P)]),
    ("lh_hmat_derive_toeplitz", C.c_int, [P, P, P, D, I32, C.POINTER(P)]),
    ("lh_hmat_clone", C.c_int, [P, P, I32, C.POINTER(P)]),
    ("lh_tree_build_strategy", C.c_int, [P, P, I64, C.c_int, C.c_int, C.c_int, C.POINTER(P)]),
    ("lh_cn2d_dense", C.c_int, [P, I64, I32, C.c_double, C.c_double, C.c_double, C.c_double, C.c_double, C.c_double, C.c_double, C.c_double, I32, P, P]),
    ("lh_hmat_spill", C.c_int, [P, P]),
    ("lh_nccl_unique_id", C.c_int, [P]),
    ("lh_nccl_init", C.c_int, [P, I32, I32, P]),
    ("lh_nccl_ready", C.c_int, [P]),
    ("lh_hmat_build_toeplitz_nccl", C.c_int, [P, P, P, P, P, I32, P, C.POINTER(P)]),
    ("lh_bcast_factors", C.c_int, [P, P, I32]),
    ("lh_hmat_resident", C.c_int, [P]),
    ("lh_hmat_destroy", None, [P]),
    ("lh_hmat_num_blocks", I64, [P]),
    ("lh_hmat_structure", C.c_int, [P, P, P]),
    ("lh_hmat_memory", C.c_int, [P, P, P]),
    ("lh_hmat_export_block", C.c_int, [P, P, I64, P, P]),
    ("lh_hmat_entry", C.c_int, [P, P, I64, I64, P]),
    ("lh_hmat_layout", C.c_int, [P, P, P]),
    ("lh_hmat_export_arena", C.c_int, [P, P, P, P, P]),
    ("lh_hmat_matvec", C.c_int, [P, P, P, I64, P, I64, I32]),
    ("lh_hlu", C.c_int, [P, P, D]),
    ("lh_solve", C.c_int, [P, P, P, I64, I32, I32]),
    ("lh_prepare_inverse", C.c_int, [P, P, D]),
    ("lh_prepare_propagator", C.c_int, [P, P, D]),
    ("lh_propagator_stats", C.c_int, [P, P]),
    ("lh_hmat_build_toeplitz_shard", C.c_int, [P, P, P, P, P, I32, I32, P]),
    ("lh_hmat_shard_pack", C.c_int, [P, P, P, I64, P]),
    ("lh_hmat_shard_unpack", C.c_int, [P, P, I32, P, I64]),
    ("lh_hmat_shard_finalize", C.c_int, [P, P]),
    ("lh_step_graph_kernels", I32, [P]),
    ("lh_cn_last_path", C.c_int, [P, P]),
    ("lh_trisolve_dense", C.c_int, [P, P, I32, I32, P, I64, I32]),
    ("lh_trisolve_block", C.c_int, [P, P, P, I32, I32, D, C.POINTER(P)]),
    ("lh_lowrank_add_recompress", C.c_int, [P, I64, I64, P, P, I32, P, P, I32, D, P, P, P]),
    ("lh_cn_steps", C.c_int, [P, P, P, P, I64, I32, I32, I32]),
    ("lh_cn_step_host", C.c_int, [P, P, P, P, P, I32]),
    ("lh_step_profile", C.c_int, [P, P, P, P, I32, I32, P]),
    ("lh_hlu_stats", C.c_int, [P, P]),
    ("lh_hmat_build_gauss_series", C.c_int, [P, P, P, P, P, P, C.c_double, C.c_double, C.c_int,
                                             C.c_double, P, P]),
    ("lh_gauss_series_terms", C.c_int, [C.c_double, C.c_double, C.c_int, C.c_double]),
    ("lh_hmat_build_gauss_series_2d", C.c_int, [P, P, P, P, P, C.c_double, C.c_double, C.c_int, C.c_double,
                                                P, P, P]),
    ("lh_gauss_cn_symbol", C.c_int, [P, C.c_int64, C.c_double, C.c_double, C.c_double, C.c_int64,
                                     C.c_double, C.c_double, C.c_double, C.c_double, P, P, P, P]),
    ("lh_pcg", C.c_int, [P, P, P, P, I64, D, I32, P, P, P, P]),
    ("lh_gmres_restarted", C.c_int, [P, P, P, P, I64, D, I32, I32, P, P, P, P]),
    ("lh_dense_gemv", C.c_int, [P, P, I64, I64, I64, P, P]),
    ("lh_hmat_save", C.c_int, [P, P, D, C.c_char_p]),
    ("lh_hmat_load", C.c_int, [P, C.c_char_p, C.POINTER(P), C.POINTER(P), C.POINTER(P), P, P]),
    ("lh_tree_points", C.c_int, [P, P]),
    ("lh_cn_symbol", C.c_int, [P, C.POINTER(MeasureC), C.POINTER(CNParamsC), P, P, P, P]),
    ("lh_frac_apply_1d", C.c_int, [P, C.POINTER(MeasureC), D, I64, I64, D, D, D, P, P, I32, P, P]),
    ("lh_frac_apply_2d", C.c_int, [P, D, D, P, D, I64, I64, D, D, D, P, P, P, P]),
    ("lh_assemble_variable_order", C.c_int, [P, I32, I64, P, P, D, D, P, P, P, P]),
]

_lib = None
_lock = threading.Lock()


def lib():
    """Load the native library (raises if it was not built)."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise ImportError(
                        f"{LIB_PATH} is missing: build it with "
                        "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback)")
                L = C.CDLL(LIB_PATH)
                for name, res, args in SIGNATURES:
                    f = getattr(L, name)
                    f.restype = res
                    f.argtypes = args
                _lib = L
    return _lib


# test / diagnostic hooks of liblevyh_b200_testing.so (include/levyh_b200_testing.h)
TESTING_SIGNATURES = [
    ("lh_debug_dump_plans", C.c_int, [P, P, C.c_int, C.c_int, D, C.c_int, C.c_int, C.c_char_p]),
    ("lh_debug_plan_timing", C.c_int, [P, P, C.c_int, C.c_int, D, C.c_int, C.c_int, C.c_int, P]),
    ("lh_debug_task_bench", C.c_int, [P, C.c_int, C.c_int, C.c_int, C.c_int, P]),
    ("lh_debug_recomp_bench", C.c_int, [P, C.c_int, C.c_int, C.c_int, C.c_int, P, P, P]),
]
TESTING_LIB_PATH = os.path.join(os.path.dirname(LIB_PATH), "liblevyh_b200_testing.so")
_testing = None


def testing():
    """The testing library (plan export, planner timing, micro-benchmarks); not product code."""
    global _testing
    if _testing is None:
        lib()  # the main library first (the testing one links against it)
        T = C.CDLL(TESTING_LIB_PATH)
        for name, res, args in TESTING_SIGNATURES:
            f = getattr(T, name)
            f.restype = res
            f.argtypes = args
        _testing = T
    return _testing


class NativeError(RuntimeError):
    pass


def check(rc, ctx=None):
    """Map an lh status code onto the reference's exception types."""
    if rc == LH_OK:
        return
    msg = lib().lh_ctx_last_error(ctx).decode() if ctx else f"native error {rc}"
    if rc == LH_EINVAL:
        raise ValueError(msg)
    if rc == LH_ESINGULAR:
        raise np.linalg.LinAlgError(msg)
    if rc == LH_ETYPE:
        raise TypeError(msg)
    if rc == LH_ENOMEM:
        raise MemoryError(msg)
    raise NativeError(f"[{rc}] {msg}")


class Context:
    """One native context per CUDA device, on torch's current stream at creation."""

    _per_device: dict = {}

    def __init__(self, device):
        import torch

        if not torch.cuda.is_available():
            raise RuntimeError("paper_1812_08324_b200 needs a CUDA device (B200); none is visible")
        self.device = device
        with torch.cuda.device(device):
            self.stream = torch.cuda.current_stream(device)
        h = C.c_void_p()
        rc = lib().lh_ctx_create(device, C.c_void_p(self.stream.cuda_stream), C.byref(h))
        self.h = h
        check(rc, h)

    @classmethod
    def get(cls, device=None):
        import torch

        if device is None:
            device = torch.cuda.current_device() if torch.cuda.is_available() else 0
        if device not in cls._per_device:
            cls._per_device[device] = Context(device)
        return cls._per_device[device]

    def sync(self):
        check(lib().lh_ctx_synchronize(self.h), self.h)

    def nccl_ready(self):
        return bool(lib().lh_nccl_ready(self.h))

    def init_nccl(self, group=None):
        """The library's own NCCL communicator over the ranks of `group` (torch.distributed,
        already initialised): rank 0 creates the unique id, the group broadcasts it, every rank
        calls lh_nccl_init.  No-op when already initialised."""
        import torch.distributed as dist

        if self.nccl_ready():
            return
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        uid = (C.c_char * 128)()
        rc0 = lib().lh_nccl_unique_id(C.cast(uid, C.c_void_p)) if rank == 0 else 0
        # a failure on rank 0 (libnccl not loadable) is broadcast too, so that no rank waits for an id
        obj = [(rc0, bytes(uid.raw)) if rank == 0 else None]
        dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group is not None else 0,
                                   group=group)
        if obj[0][0] != 0:
            raise NativeError(f"[{obj[0][0]}] rank 0 could not create the NCCL unique id (libnccl not loadable?)")
        uid = (C.c_char * 128).from_buffer_copy(obj[0][1])
        check(lib().lh_nccl_init(self.h, rank, world, C.cast(uid, C.c_void_p)), self.h)

    def torch_stream(self):
        """The library's CUDA stream as a torch stream (for CUDA-event timing)."""
        import torch

        return torch.cuda.ExternalStream(lib().lh_ctx_stream(self.h) or 0, device=self.device)


def host_ptr(a):
    return C.c_void_p(a.ctypes.data)
