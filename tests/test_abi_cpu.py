"""CPU-side checks of the C-ABI library (no GPU): it loads, exports every
symbol include/netmfp.h declares, its host-only logic is right, and compute
calls fail loudly (no CPU fallback) when no CUDA device is present."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    import __graft_entry__ as ge
    ge.build()
    from paper_2110_12782_b200 import _lib
    return _lib


def _declared():
    src = open(os.path.join(ROOT, "include", "netmfp.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(netmfp_[a-z0-9_]+)\s*\(", src)))


def test_every_declared_symbol_is_exported(L):
    lib = ctypes.CDLL(L.LIB_PATH)
    names = _declared()
    assert len(names) >= 15
    for nm in names:
        assert hasattr(lib, nm), f"{nm} not exported"
    assert set(names) == set(L.EXPORTED), "binding and header disagree"


def test_library_is_sm100a(L):
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", L.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_cheb_coeffs_host_matches_oracle(L):
    import oracle as O
    for order, mu, th in [(0, 0.2, 0.5), (10, 0.2, 0.5), (7, 0.5, 1.0)]:
        assert np.allclose(L.netmfp_cheb_coeffs(order, mu, th), O.cheb_coeffs(order, mu, th),
                           rtol=1e-12, atol=1e-13)


def test_partition_rows(L):
    from paper_2110_12782_b200 import inputs
    import oracle as O
    n, s, t = inputs.small_graph("rmat", 3000, 1, edge_factor=8)
    rp, col, deg = O.build_csr(n, s, t)
    for parts in (1, 2, 3, 8):
        b = L.netmfp_partition_rows(rp, parts)
        assert b[0] == 0 and b[-1] == n and np.all(np.diff(b) >= 0)
        cost = rp[b[1:]] - rp[b[:-1]] + np.diff(b)
        # each part within one max row cost of the ideal share
        ideal = (rp[-1] + n) / parts
        assert np.all(np.abs(cost - ideal) <= deg.max() + 1)


def test_no_cpu_fallback(L):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(L.NetmfpError) as e:
        L.Context(0, stream=0)
    assert e.value.code == L.ERR_CUDA
