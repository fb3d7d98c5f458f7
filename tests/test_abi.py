"""The C-ABI library loads and exports every symbol include/nsg.h (product interface) and
include/nsg_internal.h (measurement / test hooks) declare; the debug build exports the same; host-side
argument handling (no compute call needs a GPU here)."""
import ctypes
import os
import re

import pytest

from nsg_testutil import ROOT

HEADER = os.path.join(ROOT, "include", "nsg.h")
INTERNAL = os.path.join(ROOT, "include", "nsg_internal.h")
LIB = os.path.join(ROOT, "paper_2509_03653_b200", "libnsg.so")
DEBUG_LIB = os.path.join(ROOT, "paper_2509_03653_b200", "libnsg_debug.so")


def declared_functions(headers=(HEADER, INTERNAL)):
    names = set()
    for h in headers:
        src = re.sub(r"/\*.*?\*/", "", open(h).read(), flags=re.S)
        names |= set(re.findall(r"\b(nsg_[a-z_]+)\s*\(", src))
    return sorted(names)


def test_measurement_hooks_are_not_in_the_product_header():
    public = declared_functions((HEADER,))
    assert "nsg_window_stats_timed" not in public
    text = open(HEADER).read()
    for flag in ("NSG_FLAG_NO_FALLBACK_CHECK", "NSG_FLAG_PROFILE", "NSG_FLAG_LEGACY_FAST"):
        assert flag not in text
        assert flag in open(INTERNAL).read()


def test_debug_library_exports_the_same_symbols():
    lib = ctypes.CDLL(DEBUG_LIB)
    for name in declared_functions():
        assert hasattr(lib, name), name


def test_header_declares_expected_entry_points():
    names = declared_functions()
    for required in ("nsg_window_stats", "nsg_window_stats_packed", "nsg_workspace_bytes", "nsg_num_windows"):
        assert required in names


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(LIB)
    for name in declared_functions():
        assert hasattr(lib, name), name


def test_binding_export_list_matches_header():
    from paper_2509_03653_b200 import _lib

    assert sorted(_lib.EXPORTS) == declared_functions()


def test_no_oracle_or_gen_symbols_in_libnsg():
    lib = ctypes.CDLL(LIB)
    for name in ("nsg_oracle_window_stats_map", "nsg_oracle_window_stats_sort", "nsg_oracle_window_stats_weighted",
                 "nsg_oracle_window_distributions", "nsg_gen_host", "nsg_gen_device"):
        assert not hasattr(lib, name)


def test_product_package_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2509_03653_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in text and "from oracle" not in text, f
                assert "oracle.cpp" not in text and "nsggen" not in text, f


def test_num_windows_and_workspace():
    import paper_2509_03653_b200 as nsg

    assert nsg.num_windows(0, 5) == 0
    assert nsg.num_windows(10, 5) == 2
    assert nsg.num_windows(11, 5) == 3
    assert nsg.num_windows(1 << 23, 1 << 17) == 64
    assert nsg.workspace_bytes(0, 1 << 17) == 0
    a = nsg.workspace_bytes(1 << 17, 1 << 17)
    b = nsg.workspace_bytes(1 << 23, 1 << 17)
    assert 0 < a <= b
    assert nsg.workspace_bytes(1 << 22, 1 << 21) > 0       # L2-path-only window
    assert nsg.workspace_bytes(10, 0) == 0


def test_argument_validation_without_gpu():
    lib = ctypes.CDLL(LIB)
    lib.nsg_window_stats_packed.restype = ctypes.c_int
    lib.nsg_window_stats_packed.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_void_p,
                                            ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]
    lib.nsg_window_stats.restype = ctypes.c_int
    lib.nsg_window_stats.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint64,
                                     ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]
    # n == 0: OK, nothing launched
    assert lib.nsg_window_stats_packed(None, 0, 1 << 17, None, None, 0, None) == 0
    # NULL data with n > 0
    assert lib.nsg_window_stats_packed(None, 10, 1 << 17, 8, 256, 1 << 20, None) == 1
    assert lib.nsg_window_stats(None, None, 10, 4, 8, 256, 1 << 20, None) == 1
    # window 0 / too large
    assert lib.nsg_window_stats_packed(8, 10, 0, 8, 256, 1 << 20, None) == 1
    assert lib.nsg_window_stats_packed(8, 10, (1 << 31) + 1, 8, 256, 1 << 20, None) == 1
    # misaligned workspace / out / keys
    assert lib.nsg_window_stats_packed(8, 10, 4, 8, 255, 1 << 20, None) == 1
    assert lib.nsg_window_stats_packed(8, 10, 4, 9, 256, 1 << 20, None) == 1
    assert lib.nsg_window_stats_packed(12, 10, 4, 8, 256, 1 << 20, None) == 1


def test_from_host_argument_validation_without_gpu():
    lib = ctypes.CDLL(LIB)
    f = lib.nsg_window_stats_from_host
    f.restype = ctypes.c_int
    vp, u64 = ctypes.c_void_p, ctypes.c_uint64
    f.argtypes = [vp, u64, u64, vp, vp, vp, vp, ctypes.c_size_t, vp, vp, ctypes.c_uint32]
    # n == 0: OK, nothing launched or copied
    assert f(None, 0, 1 << 17, None, None, None, None, 0, None, None, 0) == 0
    # window 0 / too large
    assert f(8, 10, 0, 8, 8, 8, 256, 1 << 20, None, 16, 0) == 1
    assert f(8, 10, (1 << 31) + 1, 8, 8, 8, 256, 1 << 20, None, 16, 0) == 1
    # NULL host keys / staging buffer / out / copy stream; copy stream == stream
    assert f(None, 10, 4, 8, 8, 8, 256, 1 << 20, None, 16, 0) == 1
    assert f(8, 10, 4, None, 8, 8, 256, 1 << 20, None, 16, 0) == 1
    assert f(8, 10, 4, 8, None, 8, 256, 1 << 20, None, 16, 0) == 1
    assert f(8, 10, 4, 8, 8, 8, 256, 1 << 20, None, None, 0) == 1
    assert f(8, 10, 4, 8, 8, 8, 256, 1 << 20, 16, 16, 0) == 1
    # misaligned host keys / host output
    assert f(12, 10, 4, 8, 8, 8, 256, 1 << 20, None, 16, 0) == 1
    assert f(8, 10, 4, 8, 8, 12, 256, 1 << 20, None, 16, 0) == 1


def test_status_strings():
    lib = ctypes.CDLL(LIB)
    lib.nsg_status_string.restype = ctypes.c_char_p
    assert lib.nsg_status_string(0) == b"NSG_OK"
    assert lib.nsg_status_string(3) == b"NSG_ERR_WORKSPACE_TOO_SMALL"
    lib.nsg_version.restype = ctypes.c_char_p
    assert b"sm_100a" in lib.nsg_version()


def test_sass_is_sm100a():
    """The shipped library holds sm_100a SASS (cuobjdump), not PTX-only or another arch."""
    import shutil
    import subprocess

    if shutil.which("cuobjdump") is None:
        pytest.skip("cuobjdump not available")
    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_vectors_argument_validation_without_gpu():
    from paper_2509_03653_b200._lib import NsgVectors

    lib = ctypes.CDLL(LIB)
    f = lib.nsg_window_vectors
    f.restype = ctypes.c_int
    vp, u64 = ctypes.c_void_p, ctypes.c_uint64
    f.argtypes = [vp, vp, vp, u64, u64, vp, ctypes.POINTER(NsgVectors), vp, ctypes.c_size_t, vp, ctypes.c_uint32]
    ok = NsgVectors()
    # n == 0: OK, nothing launched
    assert f(None, None, None, 0, 4, None, ctypes.byref(ok), None, 0, None, 0) == 0
    # NULL vectors struct
    assert f(None, None, 8, 10, 4, 8, None, 256, 1 << 20, None, 0) == 1
    # a half-specified group
    for half in ({"link_key": 8}, {"link_packets": 8}, {"src_node": 8, "src_packets": 8},
                 {"dst_node": 8, "dst_fanin": 8}, {"src_fanout": 4}):
        v = NsgVectors(**half)
        assert f(None, None, 8, 10, 4, 8, ctypes.byref(v), 256, 1 << 20, None, 0) == 1, half
    # misaligned arrays
    for bad in ({"link_key": 12, "link_packets": 8}, {"link_key": 8, "link_packets": 6}, {"ip_sets": 4},
                {"src_node": 8, "src_packets": 8, "src_fanout": 2}):
        v = NsgVectors(**bad)
        assert f(None, None, 8, 10, 4, 8, ctypes.byref(v), 256, 1 << 20, None, 0) == 1, bad
    # input / window errors are still checked first
    assert f(None, None, None, 10, 4, 8, ctypes.byref(ok), 256, 1 << 20, None, 0) == 1
    assert f(None, None, 8, 10, 0, 8, ctypes.byref(ok), 256, 1 << 20, None, 0) == 1


def test_next_row_entry_points_validate_without_gpu():
    """Argument errors of the weighted / trace / anonymisation entry points are reported before any device
    work (so they are testable here, without a GPU)."""
    lib = ctypes.CDLL(LIB)
    vp, u64, u32, sz = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_size_t
    w = lib.nsg_window_stats_weighted
    w.restype, w.argtypes = ctypes.c_int, [vp, vp, vp, vp, u64, u64, vp, vp, sz, vp, u32]
    assert w(None, None, 8, None, 10, 4, 8, 256, 1 << 20, None, 0) == 1      # NULL n_packets
    assert w(None, None, 8, 6, 10, 4, 8, 256, 1 << 20, None, 0) == 1         # misaligned n_packets
    assert w(None, None, None, 8, 10, 4, 8, 256, 1 << 20, None, 0) == 1      # no rows
    assert w(None, None, 8, 8, 0, 4, None, None, 0, None, 0) == 0           # n == 0: nothing to do
    tw = lib.nsg_trace_workspace_bytes
    tw.restype, tw.argtypes = sz, [u64, u64, u32]
    assert tw(100, 100, 0) == 0 and tw(100, 100, 1025) == 0 and tw(100, 100, 8) > 0
    assert tw(1 << 20, 1 << 20, 1) > tw(1 << 10, 1 << 10, 1)
    tl = lib.nsg_trace_links
    tl.restype, tl.argtypes = ctypes.c_int, [vp, vp, vp, u64, u32, vp, vp, vp, vp, vp, sz, u64, u64, vp]
    assert tl(None, None, 8, 11, 1, 8, 8, 8, 8, 256, 1 << 20, 10, 10, None) == 1   # n > key_capacity
    assert tl(None, None, 8, 10, 1, None, 8, 8, 8, 256, 1 << 20, 10, 10, None) == 1  # NULL link_stats
    assert tl(None, None, 8, 10, 1, 8, 8, 8, 12, 256, 1 << 20, 10, 10, None) == 1    # misaligned rec_counts
    tn = lib.nsg_trace_nodes
    tn.restype, tn.argtypes = ctypes.c_int, [vp, u64, vp, vp, sz, u64, u64, vp]
    assert tn(8, 11, 8, 256, 1 << 20, 10, 10, None) == 1                            # m > record_capacity
    assert tn(None, 5, 8, 256, 1 << 20, 10, 10, None) == 1                          # NULL records
    tp = lib.nsg_trace_partition
    tp.restype, tp.argtypes = ctypes.c_int, [vp, vp, vp, u64, u32, vp, vp, vp, sz, u64, u64, vp]
    assert tp(None, None, 8, 10, 2, None, 8, 256, 1 << 20, 10, 10, None) == 1       # NULL send_keys
    ts = lib.nsg_trace_stats
    ts.restype, ts.argtypes = ctypes.c_int, [vp, vp, vp, u64, vp, vp, sz, vp]
    tsw = lib.nsg_trace_stats_workspace_bytes
    tsw.restype, tsw.argtypes = sz, [u64]
    assert ts(None, None, None, 0, None, None, 0, None) == 0                        # n == 0
    assert ts(None, None, 8, 10, None, 256, 1 << 30, None) == 1                     # NULL out
    assert ts(None, None, 8, 10, 8, 256, tsw(10) - 1, None) == 3                    # workspace too small
    an = lib.nsg_anonymize
    an.restype, an.argtypes = ctypes.c_int, [vp, vp, vp, u64, u64, u32, vp, vp, vp, vp, sz, vp]
    aw = lib.nsg_anonymize_workspace_bytes
    aw.restype, aw.argtypes = sz, []
    assert aw() >= (1 << 29)                                                        # the 2^32-bit bitmap
    assert an(None, None, 8, 10, 0, 1, 8, 8, None, 256, aw(), None) == 1            # NULL n_unique
    assert an(None, None, 8, 10, 0, 1, None, 8, 8, 256, aw(), None) == 1            # NULL src_out
    assert an(None, None, 8, 10, 0, 1, 8, 8, 8, 256, aw() - 1, None) == 3           # workspace too small
