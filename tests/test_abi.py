"""The C-ABI library loads and exports every symbol include/igp.h declares (no GPU needed).

Only calls that return before touching the device are made here (status strings,
version, host-side argument validation); compute calls are in the -m gpu tests.
"""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "igp.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"IGP_API\s+[\w\s\*]+?\b(igp_\w+)\s*\(", text)))


@pytest.fixture(scope="module")
def igp():
    import __graft_entry__
    __graft_entry__.build()
    import paper_2508_19737_b200 as m
    return m


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ["igp_build_graph", "igp_embed", "igp_embed_ex", "igp_embed_host", "igp_destroy_graph",
              "igp_graph_info", "igp_graph_copy_csr", "igp_philox_bits", "igp_philox_normal"]:
        assert s in syms


def test_library_exports_every_declared_symbol(igp):
    lib = ctypes.CDLL(igp.LIB_PATH)
    for s in declared_symbols():
        assert hasattr(lib, s), f"{s} declared in igp.h but not exported"
    # the binding wraps exactly the declared surface
    assert set(igp.SIGNATURES) == set(declared_symbols())


def test_only_the_abi_is_exported(igp):
    import subprocess
    out = subprocess.run(["nm", "-D", "--defined-only", igp.LIB_PATH], capture_output=True, text=True).stdout
    names = [ln.split()[-1] for ln in out.splitlines() if ln.strip()]
    text_syms = [n for n in names if not n.startswith("_") and n not in ("_init", "_fini")]
    assert all(n.startswith("igp_") for n in text_syms), text_syms


def test_host_side_calls_without_device(igp):
    lib = igp.lib()
    assert lib.igp_status_string(0) == b"IGP_OK"
    assert lib.igp_status_string(7) == b"IGP_ERR_UNSUPPORTED"
    assert b"sm_100a" in lib.igp_version()
    assert lib.igp_kernel_launch_count() == 0
    # host-validated input errors return before any device work
    h = ctypes.c_void_p()
    assert lib.igp_build_graph(None, 0, 0, None, ctypes.byref(h)) == 2
    assert lib.igp_build_graph(None, -1, 5, None, ctypes.byref(h)) == 2
    assert lib.igp_build_graph(ctypes.c_void_p(0x1000), 2**31, 5, None, ctypes.byref(h)) == 7  # not dereferenced
    assert lib.igp_build_graph(None, 0, 2**31 - 1, None, ctypes.byref(h)) == 7                # N > 2^30 - 4096
    assert lib.igp_build_graph(None, 0, 2**30 - 4095, None, ctypes.byref(h)) == 7             # just above the limit
    o = igp.make_opts(-1.0, 48, 10)
    assert lib.igp_embed_ex(None, ctypes.byref(o), None, None) == 2
    assert lib.igp_destroy_graph(None) == 0
    assert lib.igp_kernel_launch_count() == 0


def test_more_host_validated_errors(igp):
    """Argument errors that return before any device work (no GPU needed)."""
    lib = igp.lib()
    h = ctypes.c_void_p()
    assert lib.igp_build_graph_ex(None, 0, 5, 0x80, None, ctypes.byref(h)) == 2          # unknown flag
    assert lib.igp_build_graph_ex(None, 0, 5, 1 | 4, None, ctypes.byref(h)) == 2         # conflicting orders
    assert lib.igp_build_graph_ex(None, 0, 5, 4 | 8, None, ctypes.byref(h)) == 2
    assert lib.igp_build_graph_ex(None, 0, 5, 0, None, None) == 2                        # no out handle
    assert lib.igp_build_graph_ex(None, 3, 5, 0, None, ctypes.byref(h)) == 2             # edges NULL, E > 0
    assert lib.igp_graph_add_edges(None, None, 0, None) == 2
    assert lib.igp_graph_status(None) == 2
    assert lib.igp_graph_info(None, None, None, None) == 2
    assert lib.igp_graph_copy_csr(None, None, None, None, None) == 2
    assert lib.igp_destroy_graph_async(None, None) == 0
    assert lib.igp_philox_bits(0, 0, -1, None, None) == 2
    assert lib.igp_philox_normal(0, 0, 6, None, None) == 2                               # not a multiple of 4
    o = igp.make_opts(-1.0, 64, 3)
    o.flags = 0x40
    assert lib.igp_embed_host(None, 0, 4, ctypes.byref(o), None, None) == 2              # NULL h_out first
    out = (ctypes.c_float * 256)()
    assert lib.igp_embed_host(None, 0, 4, ctypes.byref(o), out, None) == 2               # unknown embed flag
    o.flags = 0
    o.eps = 0.0
    assert lib.igp_embed_host(None, 0, 4, ctypes.byref(o), out, None) == 2               # eps must be > 0
    o.eps = 1e-3
    o.ddof = 2
    assert lib.igp_embed_host(None, 0, 4, ctypes.byref(o), out, None) == 2               # ddof in {0, 1}
    o.ddof = 0
    o.d_z0 = 0x1004
    assert lib.igp_embed_host(None, 0, 4, ctypes.byref(o), out, None) == 2               # d_z0 not 16-B aligned
    assert lib.igp_birch_create(0, 0.5, 50, ctypes.byref(h)) == 2                        # BIRCH arguments
    assert lib.igp_birch_create(4, -1.0, 50, ctypes.byref(h)) == 2
    assert lib.igp_birch_create(4, 0.5, 64, ctypes.byref(h)) == 2
    assert lib.igp_birch_partial_fit(None, None, 3, None) == 2
    assert lib.igp_birch_predict_ex(None, None, 3, None, 0, None, None) == 2
    assert lib.igp_birch_destroy(None) == 0
    for bad_d in (40, 8, 2048):                                                          # multiple of 16 in [16, 1024]
        o2 = igp.make_opts(-1.0, bad_d, 3)
        assert lib.igp_embed_host(None, 0, 4, ctypes.byref(o2), out, None) == 7
    assert lib.igp_kernel_launch_count() == 0


def test_c_example_builds_against_the_header(igp):
    """examples/embed_c.c uses only include/igp.h and links libigp.so (no Python, no torch)."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("igp_build", os.path.join(ROOT, "paper_2508_19737_b200", "_build.py"))
    b = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(b)
    exe = b.build_example()
    assert os.access(exe, os.X_OK)
