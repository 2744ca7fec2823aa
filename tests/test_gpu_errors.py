"""Error behaviour of the C ABI (include/netmfp.h): invalid arguments come back
as NETMFP_ERR_ARG with a message, nothing is queued for them, and the context
stays usable — the next valid call on the same context returns the same
result as on a fresh one (deferred numeric checks and device flags of a failed
call are dropped, api.cu DevScope)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
DEV = "cuda:0"


@pytest.fixture(scope="module")
def L():
    import __graft_entry__ as ge
    ge.build()
    from paper_2110_12782_b200 import _lib
    return _lib


def padded(n, c):
    ld = (c + 31) // 32 * 32
    return torch.zeros(n, ld, dtype=torch.float32, device=DEV)[:, :c]


def _graph(L, ctx):
    from paper_2110_12782_b200 import inputs
    n, s, t = inputs.small_graph("rmat", 2048, 4, edge_factor=6)
    return L.netmfp_build_csr(ctx, n, torch.from_numpy(s).to(DEV), torch.from_numpy(t).to(DEV)), n


def test_invalid_arguments_are_reported_and_the_context_recovers(L):
    ctx = L.Context(0)
    g, n = _graph(L, ctx)
    lam = torch.zeros(40, dtype=torch.float64, device=DEV)
    # Alg. 2 needs k + s1 <= n
    with pytest.raises(L.NetmfpError) as e:
        L.netmfp_eig(ctx, g, 0.45, 40, n, 2, 3, padded(n, 40), lam)
    assert e.value.code == 1 and "k + s1" in str(e.value)
    # alpha outside (0, 0.5]
    with pytest.raises(L.NetmfpError) as e:
        L.netmfp_eig(ctx, g, 0.7, 40, 8, 2, 3, padded(n, 40), lam)
    assert e.value.code == 1
    # Omega with l < 1
    with pytest.raises(L.NetmfpError) as e:
        L.netmfp_gaussian(ctx, 1, torch.zeros(4, 0, dtype=torch.float32, device=DEV))
    assert e.value.code == 1
    # the same context still computes exactly what a fresh one does
    U1 = padded(n, 40)
    L.netmfp_eig(ctx, g, 0.45, 40, 8, 2, 3, U1, lam)
    lam1 = lam.clone()
    ctx2 = L.Context(0)
    g2, _ = _graph(L, ctx2)
    U2 = padded(n, 40)
    lam2 = torch.zeros(40, dtype=torch.float64, device=DEV)
    L.netmfp_eig(ctx2, g2, 0.45, 40, 8, 2, 3, U2, lam2)
    torch.cuda.synchronize()
    assert torch.equal(lam1, lam2) and torch.equal(U1, U2)


def test_out_of_range_vertex_ids_are_rejected(L):
    ctx = L.Context(0)
    s = torch.tensor([0, 1, 2], dtype=torch.int32, device=DEV)
    t = torch.tensor([1, 2, 7], dtype=torch.int32, device=DEV)  # 7 >= n
    with pytest.raises(L.NetmfpError) as e:
        L.netmfp_build_csr(ctx, 5, s, t)
    assert e.value.code == 1
    g = L.netmfp_build_csr(ctx, 8, s, t)  # the context is still usable
    rp, col, deg = g.export(ctx)
    assert np.array_equal(deg, [1, 2, 2, 0, 0, 0, 0, 1])
