"""ctypes binding of libhmtl_b200.so (the C ABI declared in include/hmtl_b200.h).

The library is built in-tree (paper_2506_21788_b200/libhmtl_b200.so) by
``build()`` / ``make -C paper_2506_21788_b200/csrc``.  There is no fallback:
if the library is missing or has no CUDA device, calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HMTL_LIB") or os.path.join(HERE, "libhmtl_b200.so")  # HMTL_LIB: A/B builds
CSRC = os.path.join(HERE, "csrc")

ERR_NAMES = {1: "contract", 2: "io", 3: "comm", 4: "data", 5: "config", 6: "internal"}


class HmtlError(RuntimeError):
    """hmtl::Error (hmtl/error.hpp:17-26): carries the ErrorCode."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"[{ERR_NAMES.get(code, code)}] {msg}")
        self.code = code


def build(jobs: int = 8) -> str:
    subprocess.run(["make", "-s", "-j", str(jobs), "-C", CSRC], check=True)
    return LIB_PATH


class CHyper(C.Structure):
    _fields_ = [(n, C.c_int) for n in ("n_species", "layers", "hidden", "head_width", "head_depth", "n_heads")] + [
        ("cutoff", C.c_double)
    ]


class CSpec(C.Structure):
    _fields_ = [
        ("dataset_id", C.c_int), ("n_elements", C.c_int), ("elements", C.c_uint8 * 32),
        ("n_min", C.c_int), ("n_max", C.c_int), ("alpha", C.c_double), ("sigma", C.c_double),
        ("mu", C.c_double * 20), ("count", C.c_uint64), ("structure_seed", C.c_int64),
    ]


class CSamples(C.Structure):
    _fields_ = [
        ("G", C.c_int), ("N", C.c_int), ("n_atoms", C.POINTER(C.c_int)), ("species", C.POINTER(C.c_uint8)),
        ("positions", C.POINTER(C.c_double)), ("forces", C.POINTER(C.c_double)),
        ("energy_per_atom", C.POINTER(C.c_double)), ("dataset_id", C.POINTER(C.c_uint8)),
    ]


class CCaps(C.Structure):
    _fields_ = [("max_graphs", C.c_int), ("max_nodes", C.c_int), ("max_edges", C.c_longlong)]


class CTrainCfg(C.Structure):
    _fields_ = [(n, C.c_float) for n in ("lr", "beta1", "beta2", "eps", "weight_decay", "w_energy", "w_force")] + [
        ("use_graph", C.c_int)
    ]


_P = C.c_void_p
_FP = C.POINTER(C.c_float)
_DP = C.POINTER(C.c_double)
_IP = C.POINTER(C.c_int)
_U8P = C.POINTER(C.c_uint8)

# name -> (restype, argtypes)
SIGNATURES = {
    "hmtl_abi_version": (C.c_int, []),
    "hmtl_last_error": (C.c_char_p, []),
    "hmtl_device_count": (C.c_int, []),
    "hmtl_shared_size": (C.c_size_t, [C.POINTER(CHyper)]),
    "hmtl_head_size": (C.c_size_t, [C.POINTER(CHyper)]),
    "hmtl_layout_entry": (C.c_int, [C.POINTER(CHyper), C.c_int, C.c_int, C.c_char_p, C.c_size_t,
                                    C.POINTER(C.c_size_t), C.POINTER(C.c_size_t), C.POINTER(C.c_size_t)]),
    "hmtl_init_block": (C.c_int, [C.POINTER(CHyper), C.c_uint64, C.c_int, _FP]),
    "hmtl_classify_regime": (C.c_int, [C.c_size_t, C.c_size_t, C.c_int]),
    "hmtl_memory_footprint": (C.c_size_t, [C.c_size_t, C.c_size_t, C.c_int, C.c_int]),
    "hmtl_default5_spec": (C.c_int, [C.c_int, C.POINTER(CSpec)]),
    "hmtl_generate": (C.c_int, [C.POINTER(CSpec), C.c_uint64, _IP, _IP, _IP, _U8P, _DP, _DP, _DP, _U8P]),
    "hmtl_head_placement": (C.c_int, [C.c_int, C.c_int, _DP, _DP]),
    "hmtl_ctx_create": (C.c_int, [C.c_int, C.POINTER(CHyper), C.c_uint64, _IP, C.c_int, C.POINTER(CCaps),
                                  C.POINTER(_P)]),
    "hmtl_ctx_destroy": (None, [_P]),
    "hmtl_ctx_stream": (_P, [_P]),
    "hmtl_ctx_reserve": (C.c_int, [_P, C.POINTER(CCaps)]),
    "hmtl_nbr_build": (C.c_int, [C.c_int, C.POINTER(CSamples), C.c_double, C.c_longlong, _IP, _IP, _IP, _IP, _IP,
                                 _IP]),
    "hmtl_set_block": (C.c_int, [_P, C.c_int, _FP]),
    "hmtl_get_block": (C.c_int, [_P, C.c_int, _FP]),
    "hmtl_get_grad": (C.c_int, [_P, C.c_int, _FP]),
    "hmtl_batch_upload": (C.c_int, [_P, C.POINTER(CSamples), _P]),
    "hmtl_pool_add": (C.c_int, [_P, C.POINTER(CSamples), _IP]),
    "hmtl_batch_upload_pbc": (C.c_int, [_P, C.POINTER(CSamples), C.POINTER(C.c_double), _P]),
    "hmtl_batch_edge_images": (C.c_int, [_P, _IP]),
    "hmtl_pool_bind": (C.c_int, [_P, C.c_int, _P]),
    "hmtl_build_batch": (C.c_int, [_P, _P]),
    "hmtl_batch_edges": (C.c_int, [_P, _IP, _IP, _IP, _IP]),
    "hmtl_forward": (C.c_int, [_P, _P]),
    "hmtl_predictions": (C.c_int, [_P, _FP, _FP]),
    "hmtl_loss": (C.c_int, [_P, C.c_float, C.c_float, _P]),
    "hmtl_read_loss": (C.c_int, [_P, _FP]),
    "hmtl_backward": (C.c_int, [_P, _FP, _FP, _P]),
    "hmtl_adamw": (C.c_int, [_P, C.POINTER(CTrainCfg), _P]),
    "hmtl_train_step": (C.c_int, [_P, C.POINTER(CTrainCfg), _P]),
    "hmtl_debug_fetch": (C.c_int, [_P, C.c_char_p, C.c_int, _FP, C.c_size_t, C.POINTER(C.c_size_t)]),
    "hmtl_profile_enable": (C.c_int, [_P, C.c_int]),
    "hmtl_profile_report": (C.c_int, [_P, C.c_char_p, C.c_size_t]),
    "hmtl_step_kernel_count": (C.c_int, [_P, C.POINTER(C.c_int)]),
    "hmtl_set_stream_mode": (C.c_int, [_P, C.c_int]),
    "hmtl_debug_chain_stamps": (C.c_int, [_P, C.POINTER(C.c_longlong), C.c_int]),
    "hmtl_selftest_mma_rate": (C.c_int, [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_float)]),
    "hmtl_selftest_ingress": (C.c_int, [C.c_int, C.c_int, C.c_longlong, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_float)]),
    "hmtl_selftest_pair_layout": (C.c_int, [C.c_int, C.c_int, C.POINTER(C.c_float)]),
    "hmtl_selftest_gemm": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _FP, _FP, _FP]),
    "hmtl_selftest_time": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _FP]),
    "hmtl_epoch_plan": (C.c_int, [C.c_int, _U8P, C.POINTER(C.c_uint64), C.c_int, _IP, _IP, C.c_int, C.c_uint64,
                                  C.c_int, C.c_int, _U8P, C.POINTER(C.c_uint64), C.c_size_t, _IP,
                                  C.POINTER(C.c_size_t)]),
    "hmtl_store_create": (C.c_int, [C.c_int, C.POINTER(CSamples), C.POINTER(_P)]),
    "hmtl_store_counts": (C.c_int, [_P, _U8P, C.POINTER(C.c_uint64), C.c_int, _IP]),
    "hmtl_store_bind": (C.c_int, [_P, _P, _U8P, C.POINTER(C.c_uint64), C.c_int, _P]),
    "hmtl_store_destroy": (C.c_int, [_P]),
    "hmtl_batch_shape": (C.c_int, [_P, _IP, _IP]),
    "hmtl_loss_post": (C.c_int, [_P, C.c_int, _P]),
    "hmtl_loss_wait": (C.c_int, [_P, C.c_int, C.POINTER(C.c_float)]),
    "hmtl_store_align": (C.c_int, [_P, C.c_uint8, _U8P, C.POINTER(C.c_double), C.c_int, _U8P, _IP]),
    "hmtl_align_energies": (C.c_int, [C.c_int, C.POINTER(C.c_char_p), C.c_int, C.c_uint8, C.POINTER(C.c_char_p), _U8P,
                                      C.POINTER(C.c_double), C.c_int, _U8P, _IP]),
    "hmtl_store_download": (C.c_int, [_P, _IP, _U8P, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                      C.POINTER(C.c_double), _U8P]),
    "hmtl_store_shape": (C.c_int, [_P, _IP, C.POINTER(C.c_longlong)]),
    "hmtl_shard_range": (C.c_int, [C.c_uint64, C.c_int, C.c_int, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    "hmtl_store_create_sharded": (C.c_int, [_P, C.POINTER(CSamples), _U8P, C.POINTER(C.c_uint64), _IP, _IP, C.c_int,
                                            C.POINTER(_P)]),
    "hmtl_store_fetch": (C.c_int, [_P, _P, _U8P, C.POINTER(C.c_uint64), C.c_int, _P]),
    "hmtl_store_from_hmtd": (C.c_int, [C.c_int, C.POINTER(C.c_char_p), C.c_int, C.POINTER(_P)]),
    "hmtl_hmtd_write": (C.c_int, [C.c_char_p, C.c_uint8, C.c_uint8, C.POINTER(CSamples)]),
    "hmtl_hmtd_read_header": (C.c_int, [C.c_char_p, _U8P, _U8P, C.POINTER(C.c_uint64)]),
    "hmtl_checkpoint_write": (C.c_int, [C.c_char_p, C.POINTER(CHyper), _FP, _FP, _P]),
    "hmtl_checkpoint_read_hyper": (C.c_int, [C.c_char_p, C.POINTER(CHyper), _IP]),
    "hmtl_checkpoint_save": (C.c_int, [_P, C.c_char_p, C.c_int]),
    "hmtl_checkpoint_load": (C.c_int, [_P, C.c_char_p]),
    "hmtl_comm_unique_id": (C.c_int, [_U8P]),
    "hmtl_comm_init": (C.c_int, [_P, _U8P, C.c_int, C.c_int]),
    "hmtl_comm_sync_grads": (C.c_int, [_P, _P]),
    "hmtl_comm_bytes": (C.c_int, [_P, C.POINTER(C.c_uint64)]),
    "hmtl_comm_info": (C.c_int, [_P, _IP, _IP, _IP, C.c_int]),
}

_lib = None


def lib() -> C.CDLL:
    """Load the in-tree library (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise OSError(f"{LIB_PATH} not built: run paper_2506_21788_b200._lib.build() or __graft_entry__.build()")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc != 0:
        raise HmtlError(rc, lib().hmtl_last_error().decode())
