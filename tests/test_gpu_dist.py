"""Multi-rank execution of libnetmfp on ONE GPU: two processes,
each a rank of the row-partitioned schedule, run the library's own multi-rank
code (partitioned CSR build that sorts only the rank's keys, degree
all-gather + isolated-vertex compaction of the partition, per-SpMM row
all-gathers, all-reduced Grams and sketch rows) with the host-staged
communicator (netmfp_dist_init_ops over a gloo process group).  No kernel
waits on another rank: every exchange goes through the host.  The result is
checked against the fp64 oracle's Alg. 5 and against the single-rank library
call on the same graph."""
import os
import socket

import numpy as np
import pytest

import oracle as O
from paper_2110_12782_b200 import inputs

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

PRM = dict(alpha=0.45, k=48, s1=16, q=3, T=10, b=1.0, d=24, s2=24, s3=200, z=8, prop_order=10, mu=0.2,
           theta=0.5, seed=9, logmode=0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _graph():
    # R-MAT with hubs (heavy rows) and isolated vertices (compaction)
    return inputs.small_graph("rmat", 6000, 5, edge_factor=6)


def _worker(rank, ws, port, bounds, out_dir):
    import torch.distributed as dist
    import __graft_entry__ as ge
    ge.build()
    from paper_2110_12782_b200 import _lib as L
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=ws)
    try:
        n, s, t = _graph()
        ctx = L.Context(0)
        L.netmfp_dist_init_ops(ctx, ws, rank, lambda a: dist.all_reduce(torch.from_numpy(a)),
                               lambda a, root: dist.broadcast(torch.from_numpy(a), src=root))
        dev = torch.device("cuda:0")
        g = L.netmfp_dist_build_csr(ctx, n, torch.from_numpy(s).to(dev), torch.from_numpy(t).to(dev), bounds)
        r0, ng, vol = L.netmfp_graph_rows(g)
        rp, col, deg = g.export(ctx)
        nl = int(bounds[rank + 1] - bounds[rank])
        E = torch.zeros(nl, 32, dtype=torch.float32, device=dev)[:, :PRM["d"]]
        sig = torch.zeros(PRM["d"], dtype=torch.float64, device=dev)
        lam = torch.zeros(PRM["k"], dtype=torch.float64, device=dev)
        L.netmfp_dist_stats(ctx)
        L.netmfp_embed(ctx, g, L.make_params(**PRM), E, sig, lam)
        nbytes, ncoll = L.netmfp_dist_stats(ctx)
        # the same graph on one rank (plain single-GPU call) in this process
        c1 = L.Context(0)
        g1 = L.netmfp_build_csr(c1, n, torch.from_numpy(s).to(dev), torch.from_numpy(t).to(dev))
        E1 = torch.zeros(n, 32, dtype=torch.float32, device=dev)[:, :PRM["d"]]
        s1 = torch.zeros(PRM["d"], dtype=torch.float64, device=dev)
        l1 = torch.zeros(PRM["k"], dtype=torch.float64, device=dev)
        L.netmfp_embed(c1, g1, L.make_params(**PRM), E1, s1, l1)
        np.savez(os.path.join(out_dir, f"r{rank}.npz"), r0=r0, ng=ng, vol=vol, rp=rp, col=col, deg=deg,
                 E=E.cpu().numpy(), sig=sig.cpu().numpy(), lam=lam.cpu().numpy(), nbytes=nbytes, ncoll=ncoll,
                 E1=E1.cpu().numpy()[bounds[rank]:bounds[rank + 1]], s1=s1.cpu().numpy(), l1=l1.cpu().numpy())
    finally:
        dist.destroy_process_group()


def _cols_up_to_sign(E, R, cols):
    worst = 0.0
    for j in cols:
        r = np.linalg.norm(R[:, j])
        worst = max(worst, min(np.linalg.norm(E[:, j] - R[:, j]), np.linalg.norm(E[:, j] + R[:, j])) / r)
    return worst


@pytest.mark.parametrize("split", ["balanced", "uneven"])
def test_two_ranks_on_one_gpu(tmp_path, split):
    import torch.multiprocessing as mp
    n, s, t = _graph()
    rp, col, deg = O.build_csr(n, s, t)
    assert (deg == 0).sum() > 0 and deg.max() > 64          # exercises compaction and heavy rows
    if split == "balanced":
        cost = rp + np.arange(n + 1)                          # netmfp_partition_rows' rule
        bounds = np.array([0, int(np.searchsorted(cost, cost[-1] / 2)), n], dtype=np.int64)
    else:
        bounds = np.array([0, n // 5, n], dtype=np.int64)
    mp.start_processes(_worker, args=(2, _free_port(), bounds, str(tmp_path)), nprocs=2, join=True,
                       start_method="spawn")
    parts = [dict(np.load(os.path.join(tmp_path, f"r{r}.npz"))) for r in range(2)]
    # partitioned CSR: bit-exact slices with global column ids, vol(G) all-reduced
    for r, p in enumerate(parts):
        b0, b1 = bounds[r], bounds[r + 1]
        assert p["r0"] == b0 and p["ng"] == n and p["vol"] == col.size
        assert np.array_equal(p["rp"], rp[b0:b1 + 1] - rp[b0])
        assert np.array_equal(p["col"], col[rp[b0]:rp[b1]])
        assert np.array_equal(p["deg"], deg[b0:b1])
        assert p["ncoll"] > 0 and p["nbytes"] > 0
    ref = O.netmf_plus(n, s, t, **PRM)
    E = np.concatenate([p["E"] for p in parts], axis=0).astype(np.float64)
    E1 = np.concatenate([p["E1"] for p in parts], axis=0).astype(np.float64)
    for p in parts:
        # replicated results identical on both ranks; oracle parity
        assert np.array_equal(p["lam"], parts[0]["lam"]) and np.array_equal(p["sig"], parts[0]["sig"])
        assert np.abs(p["lam"] - ref["lam"]).max() <= 1e-3 * abs(ref["lam"][0])
        so = ref["sigma"]
        lead = so >= 1e-2 * so[0]
        assert np.abs(p["sig"] - so)[lead].max() <= 1e-3 * so[0]
        # the single-rank library call on the same graph
        assert np.abs(p["lam"] - p["l1"]).max() <= 1e-5 * abs(p["l1"][0])
        assert np.abs(p["sig"] - p["s1"]).max() <= 1e-4 * p["s1"][0]
    assert np.all(E[deg == 0] == 0.0)                        # isolated vertices [R2]
    so = ref["sigma"]
    cols = [j for j in range(8) if (j == 0 or so[j - 1] - so[j] > 1e-2 * so[j]) and so[j] - so[j + 1] > 1e-2 * so[j]]
    assert cols
    assert _cols_up_to_sign(E, ref["E"], cols) <= 1e-3
    assert _cols_up_to_sign(E, E1, cols) <= 1e-4


def _nccl_worker(rank, ws, port, bounds, out_dir):
    """One rank per GPU over the library's own NCCL communicator (netmfp_dist_init):
    the row-partitioned path exactly as `bench.py --gpus N` runs it."""
    import torch.distributed as dist
    import __graft_entry__ as ge
    ge.build()
    from paper_2110_12782_b200 import _lib as L
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=ws)
    try:
        torch.cuda.set_device(rank)
        dev = torch.device(f"cuda:{rank}")
        uid = [L.netmfp_dist_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        ctx = L.Context(rank)
        L.netmfp_dist_init(ctx, uid[0], ws, rank)
        n, s, t = _graph()
        g = L.netmfp_dist_build_csr(ctx, n, torch.from_numpy(s).to(dev), torch.from_numpy(t).to(dev), bounds)
        nl = int(bounds[rank + 1] - bounds[rank])
        E = torch.zeros(nl, 32, dtype=torch.float32, device=dev)[:, :PRM["d"]]
        sig = torch.zeros(PRM["d"], dtype=torch.float64, device=dev)
        lam = torch.zeros(PRM["k"], dtype=torch.float64, device=dev)
        L.netmfp_embed(ctx, g, L.make_params(**PRM), E, sig, lam)
        torch.cuda.synchronize(dev)
        np.savez(os.path.join(out_dir, f"n{rank}.npz"), E=E.cpu().numpy(), sig=sig.cpu().numpy(),
                 lam=lam.cpu().numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                    reason="the NCCL row-partitioned path needs two GPUs (one rank per GPU)")
def test_two_ranks_nccl_on_two_gpus(tmp_path):
    """The library's NCCL communicator with one rank per GPU: oracle parity of
    Alg. 5 on the row-partitioned graph (replicated λ, σ identical on both
    ranks; E's separated columns up to sign)."""
    import torch.multiprocessing as mp
    n, s, t = _graph()
    rp, col, deg = O.build_csr(n, s, t)
    cost = rp + np.arange(n + 1)
    bounds = np.array([0, int(np.searchsorted(cost, cost[-1] / 2)), n], dtype=np.int64)
    mp.start_processes(_nccl_worker, args=(2, _free_port(), bounds, str(tmp_path)), nprocs=2, join=True,
                       start_method="spawn")
    parts = [dict(np.load(os.path.join(tmp_path, f"n{r}.npz"))) for r in range(2)]
    ref = O.netmf_plus(n, s, t, **PRM)
    so = ref["sigma"]
    lead = so >= 1e-2 * so[0]
    for p in parts:
        assert np.array_equal(p["lam"], parts[0]["lam"]) and np.array_equal(p["sig"], parts[0]["sig"])
        assert np.abs(p["lam"] - ref["lam"]).max() <= 1e-3 * abs(ref["lam"][0])
        assert np.abs(p["sig"] - so)[lead].max() <= 1e-3 * so[0]
    E = np.concatenate([p["E"] for p in parts], axis=0).astype(np.float64)
    assert np.all(E[deg == 0] == 0.0)
    cols = [j for j in range(8) if (j == 0 or so[j - 1] - so[j] > 1e-2 * so[j]) and so[j] - so[j + 1] > 1e-2 * so[j]]
    assert _cols_up_to_sign(E, ref["E"], cols) <= 1e-3
