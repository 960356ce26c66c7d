"""ctypes binding of libsdb.so — the C-ABI declared in include/sdb_api.h.

The library is built in-tree (``make -C paper_2407_02031_b200/csrc`` or
``__graft_entry__.build()``).  There is no fallback: if the shared library is
missing, or no sm_100 device is visible when a kernel is called, the call
raises.  Loading the library itself needs no GPU (the CPU test-suite checks
the exported symbols).
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "libsdb.so"

SDB_OK = 0
SDB_EINVAL = -1
SDB_ECUDA = -2
SDB_EUNSUP = -3

SDB_F32 = 0
SDB_BF16 = 1
SDB_F16 = 2

#: every symbol include/sdb_api.h declares (checked by tests/test_abi.py)
EXPORTED = (
    "sdb_version",
    "sdb_last_error",
    "sdb_device_ok",
    "sdb_lora_plan",
    "sdb_lora_patch",
    "sdb_lora_patch_one",
    "sdb_groupnorm_workspace",
    "sdb_groupnorm_silu",
    "sdb_residual_inject",
    "sdb_residual_inject_bias",
    "sdb_residual_inject_gn",
    "sdb_groupnorm_apply",
    "sdb_cfg_ddim_step",
    "sdb_conv_out",
    "sdb_groupnorm_set_mode",
    "sdb_groupnorm_launches",
    "sdb_groupnorm_stream_plan",
    "sdb_groupnorm_resident_plan",
    "sdb_set_pdl",
)


class LoraJob(ctypes.Structure):
    """Mirror of ``sdb_lora_job`` (include/sdb_api.h)."""

    _fields_ = [
        ("w_in", ctypes.c_void_p),
        ("w_out", ctypes.c_void_p),
        ("down", ctypes.c_void_p),
        ("up", ctypes.c_void_p),
        ("h1", ctypes.c_int64),
        ("h2", ctypes.c_int64),
        ("ldw", ctypes.c_int64),
        ("ldd", ctypes.c_int64),
        ("ldu", ctypes.c_int64),
        ("rank", ctypes.c_int32),
        ("scale", ctypes.c_float),
        ("tile_begin", ctypes.c_int64),
    ]


class SdbError(RuntimeError):
    """A C-ABI call returned a non-zero status."""

    def __init__(self, func: str, code: int, message: str):
        super().__init__(f"{func} failed ({code}): {message}")
        self.code = code
        self.message = message


_lib = None


def _declare(lib: ctypes.CDLL) -> None:
    vp, i64, i32, f32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_float
    lib.sdb_version.restype = ctypes.c_char_p
    lib.sdb_version.argtypes = []
    lib.sdb_last_error.restype = ctypes.c_char_p
    lib.sdb_last_error.argtypes = []
    lib.sdb_device_ok.restype = i32
    lib.sdb_device_ok.argtypes = [i32]
    lib.sdb_lora_plan.restype = i32
    lib.sdb_lora_plan.argtypes = [ctypes.POINTER(LoraJob), i32, i32, i32,
                                  ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int)]
    lib.sdb_lora_patch.restype = i32
    lib.sdb_lora_patch.argtypes = [vp, i32, i64, i32, i32, i32, f32, i32, vp]
    lib.sdb_lora_patch_one.restype = i32
    lib.sdb_lora_patch_one.argtypes = [vp, vp, i64, i64, i64, vp, i64, vp, i64, ctypes.c_int32,
                                       f32, f32, i32, i32, vp]
    lib.sdb_groupnorm_workspace.restype = ctypes.c_size_t
    lib.sdb_groupnorm_workspace.argtypes = [i64, i64, i64, i64]
    lib.sdb_groupnorm_silu.restype = i32
    lib.sdb_groupnorm_silu.argtypes = [vp, vp, vp, vp, vp, i64, i64, i64, i64, f32, i32, i32, vp, vp]
    lib.sdb_groupnorm_apply.restype = i32
    lib.sdb_groupnorm_apply.argtypes = [vp, vp, vp, vp, vp, i64, i64, i64, i64, f32, i32, i32, vp, vp]
    lib.sdb_residual_inject_gn.restype = i32
    lib.sdb_residual_inject_gn.argtypes = [vp, vp, vp, ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_float),
                                           i32, i64, i64, i64, i64, vp, vp, i64, vp, i32, vp]
    lib.sdb_residual_inject.restype = i32
    lib.sdb_residual_inject.argtypes = [vp, vp, vp, ctypes.POINTER(ctypes.c_void_p),
                                        ctypes.POINTER(ctypes.c_float), i32, i64, i64, i64, i32, vp]
    lib.sdb_residual_inject_bias.restype = i32
    lib.sdb_residual_inject_bias.argtypes = [vp, vp, vp, ctypes.POINTER(ctypes.c_void_p),
                                             ctypes.POINTER(ctypes.c_float), i32, i64, i64, i64, vp, vp, i32, vp]
    lib.sdb_cfg_ddim_step.restype = i32
    lib.sdb_cfg_ddim_step.argtypes = [vp, i32, vp, vp, vp, i32, i64, vp, vp, vp]
    lib.sdb_groupnorm_set_mode.restype = None
    lib.sdb_groupnorm_set_mode.argtypes = [i32]
    lib.sdb_groupnorm_launches.restype = i32
    lib.sdb_groupnorm_launches.argtypes = [i64, i64, i64, i64, i32]
    lib.sdb_set_pdl.restype = i32
    lib.sdb_set_pdl.argtypes = [i32]
    lib.sdb_groupnorm_stream_plan.restype = i32
    lib.sdb_groupnorm_stream_plan.argtypes = [i64, i64, i64, i64, ctypes.POINTER(ctypes.c_int)]
    lib.sdb_groupnorm_resident_plan.restype = i32
    lib.sdb_groupnorm_resident_plan.argtypes = [i64, i64, i64, i64, ctypes.POINTER(ctypes.c_int)]
    lib.sdb_conv_out.restype = i32
    lib.sdb_conv_out.argtypes = [vp, vp, vp, vp, i64, i64, i64, i64, i64, i32, vp]


def lib() -> ctypes.CDLL:
    """Load (once) and return the C-ABI library; raise if it was not built."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `make -C {LIB_PATH.parent / 'csrc'}` "
                "or __graft_entry__.build(); there is no CPU fallback")
        handle = ctypes.CDLL(str(LIB_PATH), mode=os.RTLD_NOW | getattr(os, "RTLD_GLOBAL", 0))
        _declare(handle)
        _declare_tc(handle)
        _lib = handle
    return _lib


def check(func: str, rc: int) -> None:
    if rc != SDB_OK:
        msg = lib().sdb_last_error().decode(errors="replace")
        raise SdbError(func, rc, msg)


def last_error() -> str:
    return lib().sdb_last_error().decode(errors="replace")


def version() -> str:
    return lib().sdb_version().decode()


class LoraTcJob(ctypes.Structure):
    """Mirror of ``sdb_lora_tc_job`` (include/sdb_api.h)."""

    _fields_ = [
        ("w_in", ctypes.c_void_p),
        ("w_out", ctypes.c_void_p),
        ("h1", ctypes.c_int64),
        ("h2", ctypes.c_int64),
        ("ldw", ctypes.c_int64),
        ("a_packed", ctypes.c_void_p),
        ("b_packed", ctypes.c_void_p),
        ("rank", ctypes.c_int32),
        ("scale", ctypes.c_float),
        ("lo_mask", ctypes.c_int32),
    ]


class LoraSrc(ctypes.Structure):
    """Mirror of ``sdb_lora_src`` (include/sdb_api.h)."""

    _fields_ = [
        ("down", ctypes.c_void_p),
        ("ldd", ctypes.c_int64),
        ("up", ctypes.c_void_p),
        ("ldu", ctypes.c_int64),
        ("rank", ctypes.c_int32),
        ("scale", ctypes.c_float),
    ]


EXPORTED = EXPORTED + ("sdb_lora_pack_bytes", "sdb_lora_pack", "sdb_lora_pack_multi", "sdb_lora_pack_multi_layout",
                       "sdb_lora_tc_plan",
                       "sdb_lora_tc_patch", "sdb_lora_tc_set_mode", "sdb_geglu", "sdb_ff_geglu", "sdb_add_layernorm",
                       "sdb_cross_attention", "sdb_stream_wait_value32", "sdb_stream_write_value32",
                       "sdb_memcpy_async", "sdb_cross_attention_set_mode", "sdb_self_attention",
                       "sdb_upsample2x", "sdb_batched_copy", "sdb_batched_copy_chunk_vectors")


def _declare_tc(lib: ctypes.CDLL) -> None:
    vp, i64, i32, f32, sz = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_float, ctypes.c_size_t
    lib.sdb_lora_pack_bytes.restype = i32
    lib.sdb_lora_pack_bytes.argtypes = [i64, i64, ctypes.c_int32, ctypes.POINTER(sz), ctypes.POINTER(sz)]
    lib.sdb_lora_pack.restype = i32
    lib.sdb_lora_pack.argtypes = [vp, i64, vp, i64, i64, i64, ctypes.c_int32, vp, vp, vp]
    lib.sdb_lora_pack_multi.restype = i32
    lib.sdb_lora_pack_multi.argtypes = [ctypes.POINTER(LoraSrc), i32, i64, i64, vp, vp, vp]
    lib.sdb_lora_pack_multi_layout.restype = i32
    lib.sdb_lora_pack_multi_layout.argtypes = [ctypes.POINTER(LoraSrc), i32, i64, i64, ctypes.POINTER(sz),
                                               ctypes.POINTER(sz), ctypes.POINTER(ctypes.c_float),
                                               ctypes.POINTER(ctypes.c_int32)]
    lib.sdb_lora_tc_plan.restype = i32
    lib.sdb_lora_tc_plan.argtypes = [ctypes.POINTER(LoraTcJob), i32, vp, sz, ctypes.POINTER(sz),
                                     ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)]
    lib.sdb_lora_tc_patch.restype = i32
    lib.sdb_lora_tc_patch.argtypes = [vp, i32, i32, i32, i32, f32, i32, vp]
    lib.sdb_lora_tc_set_mode.restype = i32
    lib.sdb_lora_tc_set_mode.argtypes = [i32]
    lib.sdb_batched_copy.restype = i32
    lib.sdb_batched_copy.argtypes = [vp, vp, vp, vp, i32, i64, vp]
    lib.sdb_batched_copy_chunk_vectors.restype = i64
    lib.sdb_batched_copy_chunk_vectors.argtypes = []
    lib.sdb_upsample2x.restype = i32
    lib.sdb_upsample2x.argtypes = [vp, vp, i64, i64, i64, i64, i32, vp]
    lib.sdb_geglu.restype = i32
    lib.sdb_geglu.argtypes = [vp, vp, i64, i64, i32, vp]
    lib.sdb_stream_wait_value32.restype = i32
    lib.sdb_stream_wait_value32.argtypes = [vp, vp, ctypes.c_uint32]
    lib.sdb_stream_write_value32.restype = i32
    lib.sdb_stream_write_value32.argtypes = [vp, vp, ctypes.c_uint32]
    lib.sdb_self_attention.restype = i32
    lib.sdb_self_attention.argtypes = [vp, i64, vp, i64, i32, i32, i32, i32, f32, i32, vp]
    lib.sdb_cross_attention_set_mode.restype = i32
    lib.sdb_cross_attention_set_mode.argtypes = [i32]
    lib.sdb_memcpy_async.restype = i32
    lib.sdb_memcpy_async.argtypes = [vp, vp, ctypes.c_size_t, vp]
    lib.sdb_cross_attention.restype = i32
    lib.sdb_cross_attention.argtypes = [vp, i64, vp, i64, i64, vp, i64, i32, i32, i32, i32, i32, f32, i32, vp]
    lib.sdb_ff_geglu.restype = i32
    lib.sdb_ff_geglu.argtypes = [vp, vp, vp, vp, i64, i64, i64, vp]
    lib.sdb_add_layernorm.restype = i32
    lib.sdb_add_layernorm.argtypes = [vp, vp, vp, vp, vp, i64, i64, f32, i32, vp]
