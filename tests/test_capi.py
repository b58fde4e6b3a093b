"""The C-ABI library loads and exports every entry point include/alto_b200.h
declares (no device work: safe without a GPU)."""

import ctypes
import re
from pathlib import Path

from paper_2403_06348_b200 import _native as nat

HEADER = Path(__file__).resolve().parent.parent / "include" / "alto_b200.h"


def declared():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:int|const char \*)\s*(alto_\w+)\s*\(", text, re.M)))


def test_header_declares_entry_points():
    names = declared()
    for core in ("alto_encode", "alto_sort_pairs", "alto_partition", "alto_mttkrp_stream",
                 "alto_mttkrp_exact", "alto_mttkrp_oriented", "alto_phi_stream", "alto_phi_oriented",
                 "alto_phi_exact", "alto_pi", "alto_apr_update", "alto_loglik"):
        assert core in names


def test_library_exports_every_declared_symbol():
    lib = nat.load()
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_covers_header():
    assert set(declared()) <= set(nat.EXPORTED)


def test_host_only_calls():
    lib = nat.load()
    assert lib.alto_abi_version() == 1
    b = ctypes.c_size_t(0)
    assert lib.alto_run_scratch_bytes(1000, ctypes.byref(b)) == 0 and b.value > 1000 * 16
    n = ctypes.c_int64(0)
    assert lib.alto_default_segments(1_000_000, ctypes.byref(n)) == 0 and n.value >= 1


def test_struct_sizes_match_c_layout():
    # alto_layout_t: 4 int32 + 16 int64 + 17 int32 + 4*192 uint8 (+ padding)
    assert ctypes.sizeof(nat.LayoutStruct) >= 16 + 128 + 68 + 768
    assert nat.LayoutStruct.dims.offset == 16
    assert ctypes.sizeof(nat.FactorsStruct) == 8 + 16 * 8 + 16 * 8


def test_nccl_entries_resolve_without_a_gpu():
    """NCCL is resolved at run time (csrc/comm.cu): the version and a unique
    id need no device; creating a communicator without one is a
    RuntimeError (ALTO_ERR_CUDA), not a crash."""
    import pytest
    import torch

    lib = nat.load()
    v = ctypes.c_int32(0)
    assert lib.alto_nccl_version(ctypes.byref(v)) == 0 and v.value >= 21800
    uid = (ctypes.c_uint8 * 128)()
    assert lib.alto_nccl_unique_id(ctypes.cast(uid, ctypes.c_void_p), 128) == 0
    assert any(bytes(uid))
    assert lib.alto_nccl_unique_id(ctypes.cast(uid, ctypes.c_void_p), 16) == 1  # too short: ValueError
    if torch.cuda.is_available():
        pytest.skip("a GPU is present: the communicator would be created")
    from paper_2403_06348_b200 import distributed as D

    with pytest.raises(RuntimeError, match="ncclCommInitRank"):
        D.NativeComm()
