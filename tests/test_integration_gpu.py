"""INTEGRATION.md's FFI-level binding is executable: the ctypes snippet a
maintainer would add to the reference's qtape/_native.py (_load_b200 +
conv_forward_b200) is extracted from the document, run against the in-tree
libqtape_b200.so, and matches the oracle's conv forward (the reference's
fixed-order C kernel, _kernels.c:10-51, where compiled)."""

import os
import re

import numpy as np
import pytest

import oracle as O
from gpu_util import CONV_TOL, norm_err

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _snippet():
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    blocks = re.findall(r"```python\n(.*?)```", text, re.S)
    code = [b for b in blocks if "def conv_forward_b200" in b]
    assert code, "INTEGRATION.md lost its FFI snippet"
    return code[0]


@pytest.mark.parametrize("shape", [(2, 16, 16, 32, 3, 1, 1), (2, 3, 9, 4, 3, 1, 1),
                                   (4, 64, 8, 256, 1, 1, 0), (2, 32, 16, 32, 2, 2, 0)])
def test_integration_snippet_runs(shape, monkeypatch):
    from paper_1901_07988_b200 import _native as N
    monkeypatch.setenv("QTAPE_B200_LIB", N.library_path())
    ns = {}
    exec(compile(_snippet(), "INTEGRATION.md", "exec"), ns)
    n, ci, h, co, k, s, p = shape
    rng = np.random.default_rng(sum(shape))
    x = rng.standard_normal((n, ci, h, h)).astype(np.float32)
    w = (rng.standard_normal((co, ci, k, k)) * 0.2).astype(np.float32)
    got = ns["conv_forward_b200"](x, w, s, p)
    want = O.conv_fwd(x, w, s, p)
    assert got.shape == want.shape
    assert norm_err(got, want) < CONV_TOL
