"""The C-ABI library loads and exports every symbol include/qtape_b200.h
declares (no compute: this runs on the CPU-only build container)."""

import ctypes
import os
import re

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "qtape_b200.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(qt_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_entry_points():
    syms = declared_symbols()
    for must in ("qt_quantize_pack", "qt_unpack_dequant", "qt_bn_relu_forward", "qt_bn_stats",
                 "qt_conv_forward", "qt_conv_dgrad", "qt_conv_wgrad", "qt_bn_backward_reduce",
                 "qt_bn_backward_apply", "qt_softmax_xent", "qt_sgd", "qt_matmul"):
        assert must in syms


def test_library_exports_every_declared_symbol():
    from paper_1901_07988_b200 import _native as N
    lib = N.lib()
    for s in declared_symbols():
        assert hasattr(lib, s), s
        assert s in N.SIGNATURES, f"{s} has no ctypes signature"
    raw = ctypes.CDLL(N.library_path())
    for s in declared_symbols():
        getattr(raw, s)


def test_host_queries_without_gpu():
    from paper_1901_07988_b200 import _native as N
    assert N.lib().qt_version() >= 10000
    assert N.query("qt_bn_stats_workspace", 128, 64, 1024) > 0
    assert N.query("qt_bn_backward_workspace", 128, 64, 1024) > 0
    assert N.query("qt_conv_wgrad_workspace", 128, 16, 32, 32, 16, 3, 3, 1, 1) > 0
    assert N.lib().qt_error_string(-1) == b"invalid argument"


def test_concurrent_backward_setter_returns_previous():
    """qt_set_concurrent_backward is a host-side flag (no GPU needed)."""
    from paper_1901_07988_b200 import _native as N
    prev = N.query("qt_set_concurrent_backward", 1)
    try:
        assert N.query("qt_set_concurrent_backward", 1) == 1
        assert N.query("qt_set_concurrent_backward", 0) == 1
        assert N.query("qt_set_concurrent_backward", 0) == 0
    finally:
        N.query("qt_set_concurrent_backward", prev)


def test_built_for_sm100a():
    import subprocess
    from paper_1901_07988_b200 import _native as N
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", N.library_path()],
                         capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_no_cpu_fallback_path():
    """The product package never imports the oracle."""
    pkg = os.path.join(ROOT, "paper_1901_07988_b200")
    for fn in os.listdir(pkg):
        if fn.endswith(".py"):
            assert "oracle" not in re.sub(r"#.*", "", open(os.path.join(pkg, fn)).read()
                                          ).replace("oracle/", ""), fn
