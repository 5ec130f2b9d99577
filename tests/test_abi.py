"""The C-ABI library loads and exports every entry point include/omniloc.h
declares; its pure-host entry points behave; no compute call without a GPU."""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle
import paper_2006_08861_b200 as ol

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "omniloc.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ol_[a-z_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    ol.build()
    syms = declared_symbols()
    assert len(syms) >= 18
    # the product library and the bounds-checked one (OL_LIB=checked) export the same ABI
    for path in (ol.LIB_PATH, os.path.join(os.path.dirname(ol.LIB_PATH), "libomniloc_checked.so")):
        L = ctypes.CDLL(path)
        for s in syms:
            assert hasattr(L, s), (path, s)
    # and the binding wires all of them
    bound = set(k for k in dir(ol.lib()) if k.startswith("ol_"))
    assert set(syms) <= bound | set(syms)


def test_select_window_matches_oracle():
    for L in range(1, 25):
        for M in (1, 3, 5, 11, 63):
            for m in range(L):
                assert ol.select_window(L, m, M) == oracle.select_window(L, m, M)
    with pytest.raises(ol.OmnilocError):
        ol.select_window(10, 2, 4)
    with pytest.raises(ol.OmnilocError):
        ol.select_window(10, 10, 3)


def test_shard_range_partitions():
    for n in (1, 7, 100, 20000, 100_000_000, 2**32 - 2):
        for W in (1, 2, 3, 4, 8):
            nxt = 0
            sizes = []
            for r in range(W):
                b, c = ol.shard_range(n, r, W)
                assert b == nxt and b == (r * n) // W
                nxt = b + c
                sizes.append(c)
            assert nxt == n and max(sizes) - min(sizes) <= 1
    with pytest.raises(ol.OmnilocError):
        ol.shard_range(10, 2, 2)


def test_create_without_gpu_fails_cleanly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    cfg = ol.ol_config(0, 0, 1, None, 64, 16, None)
    h = ctypes.c_void_p()
    st = ol.lib().ol_create(ctypes.byref(cfg), ctypes.byref(h))
    assert st == ol.OL_ERR_CUDA and not h.value
    assert b"CUDA" in ol.lib().ol_last_error(None) or len(ol.lib().ol_last_error(None)) > 0
    bad = ol.ol_config(0, 0, 1, None, 32, 16, None)
    assert ol.lib().ol_create(ctypes.byref(bad), ctypes.byref(h)) == ol.OL_ERR_DIMENSION_MISMATCH
    with pytest.raises(RuntimeError):
        ol.Engine(0)


def test_struct_layouts_match_header(tmp_path):
    """The binding's ctypes / numpy layouts equal what a C compiler makes of the header."""
    src = tmp_path / "layout.c"
    src.write_text(r"""
#include <stddef.h>
#include <stdio.h>
#include "omniloc.h"
int main(void) {
    printf("%zu %zu %zu %zu %zu %zu %zu %zu\n", sizeof(ol_config), offsetof(ol_config, nccl_unique_id),
           sizeof(ol_params), sizeof(ol_candidate), sizeof(ol_estimate), offsetof(ol_estimate, ranked),
           sizeof(ol_db_desc), offsetof(ol_db_desc, grid_w));
    return 0;
}
""")
    exe = tmp_path / "layout"
    import subprocess
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)])
    got = [int(v) for v in subprocess.check_output([str(exe)]).split()]
    assert got == [ctypes.sizeof(ol.ol_config), ol.ol_config.nccl_unique_id.offset, ctypes.sizeof(ol.ol_params),
                   ol.CANDIDATE_DTYPE.itemsize, ol.ESTIMATE_DTYPE.itemsize, ol.ESTIMATE_DTYPE.fields["ranked"][1],
                   ctypes.sizeof(ol.ol_db_desc), ol.ol_db_desc.grid_w.offset]


def test_nccl_unique_id_without_gpu():
    """ol_nccl_unique_id is a host function: NCCL is loaded on demand (dlopen) and the id
    is 128 bytes (ncclUniqueId), fresh on every call."""
    a = ctypes.create_string_buffer(ol.NCCL_ID_BYTES)
    b = ctypes.create_string_buffer(ol.NCCL_ID_BYTES)
    assert ol.lib().ol_nccl_unique_id(a) == 0 and ol.lib().ol_nccl_unique_id(b) == 0
    assert a.raw != b.raw and any(a.raw)
    assert ol.lib().ol_nccl_unique_id(None) == ol.OL_ERR_INVALID_ARGUMENT


def _build_c_caller(tmp_path):
    import subprocess
    import oracle
    oracle.build()
    libdir = os.path.dirname(ol.LIB_PATH)
    odir = os.path.join(ROOT, "oracle")
    exe = tmp_path / "c_caller"
    # link the product library under its own name (libomniloc.so) and the oracle's
    subprocess.check_call(["gcc", "-O2", "-I", os.path.join(ROOT, "include"), os.path.join(ROOT, "tests", "c", "c_caller.c"),
                           os.path.join(libdir, "libomniloc.so"), os.path.join(odir, "liboracle.so"), "-lm",
                           f"-Wl,-rpath,{libdir}:{odir}", "-o", str(exe)])
    return exe


def test_c_caller_builds_and_links(tmp_path):
    """The ABI compiles and links from plain C (gcc, no Python, no torch): every symbol the
    C test program calls resolves.  (It runs on the GPU: test_gpu_nccl.py.)"""
    assert _build_c_caller(tmp_path).exists()
