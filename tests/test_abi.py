"""The C-ABI library builds, loads without a GPU and exports every symbol
include/sdb_api.h declares (no compute calls here)."""

import ctypes
import re
from pathlib import Path

from paper_2407_02031_b200 import _lib

ROOT = Path(__file__).resolve().parent.parent


def header_symbols():
    text = (ROOT / "include" / "sdb_api.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\*?\s+\*?(sdb_[a-z_0-9]+)\(", text, re.M)))


def test_header_matches_binding_list():
    assert header_symbols() == sorted(_lib.EXPORTED)


def test_library_exports_every_declared_symbol():
    lib = _lib.lib()
    for name in header_symbols():
        assert hasattr(lib, name), name


def test_version_and_error_channel():
    assert "sm_100a" in _lib.version()
    assert isinstance(_lib.last_error(), str)


def test_job_struct_layout_matches_header():
    # 4 pointers, 5 int64, int32 + float, int64 -> 88 bytes, 8-byte aligned
    assert ctypes.sizeof(_lib.LoraJob) == 88
    assert _lib.LoraJob.tile_begin.offset == 80


def test_plan_is_host_only_and_validates():
    lib = _lib.lib()
    jobs = (_lib.LoraJob * 2)()
    for j, (h1, h2) in zip(jobs, [(320, 36), (1280, 1280)]):
        j.w_in = j.w_out = j.down = j.up = 0x1000
        j.h1, j.h2, j.ldw, j.ldd, j.ldu, j.rank, j.scale = h1, h2, h2, 8, h2, 8, 1.0
    total, path = ctypes.c_int64(0), ctypes.c_int(-1)
    rc = lib.sdb_lora_plan(jobs, 2, _lib.SDB_BF16, _lib.SDB_BF16, ctypes.byref(total), ctypes.byref(path))
    assert rc == 0
    assert jobs[0].tile_begin == 0 and jobs[1].tile_begin > 0
    assert total.value > jobs[1].tile_begin
    jobs[1].rank = 0
    rc = lib.sdb_lora_plan(jobs, 2, _lib.SDB_BF16, _lib.SDB_BF16, ctypes.byref(total), ctypes.byref(path))
    assert rc == _lib.SDB_EINVAL
    assert "rank" in _lib.last_error()


def test_groupnorm_workspace_query_is_host_only():
    assert _lib.lib().sdb_groupnorm_workspace(2, 128 * 128, 320, 32) > 0
    assert _lib.lib().sdb_groupnorm_workspace(0, 1, 8, 1) == 0
