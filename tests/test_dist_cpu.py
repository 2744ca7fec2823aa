"""world_size-2 gloo test of the row-partitioned schedule: the
collectives at the points where the CUDA library issues NCCL calls reproduce
the single-process oracle (λ, σ exactly up to fp64 rounding, E up to the
column signs of the SVD)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_2110_12782_b200 import inputs

PRM = dict(alpha=0.45, k=12, s1=6, q=2, T=5, b=1.0, d=6, s2=6, s3=20, z=4, prop_order=4, mu=0.2, theta=0.5,
           seed=11, logmode=0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, n, src, dst, bounds, out_dir):
    from tests._dist_ref import dist_netmf_plus
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=ws)
    try:
        r = dist_netmf_plus(n, src, dst, bounds, **PRM)
        np.savez(os.path.join(out_dir, f"r{rank}.npz"), **r)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("balanced", [True, False])
def test_row_partitioned_schedule_matches_oracle(tmp_path, balanced):
    n, s, t = inputs.small_graph("rmat", 300, 7, edge_factor=6)
    rp, col, deg = O.build_csr(n, s, t)
    if balanced:
        cost = rp + np.arange(n + 1)                 # the library's netmfp_partition_rows rule
        bounds = np.array([0] + [int(np.searchsorted(cost, cost[-1] * r / 2)) for r in (1,)] + [n])
    else:
        bounds = np.array([0, n // 3, n])
    port = _free_port()
    mp.start_processes(_worker, args=(2, port, n, s, t, bounds, str(tmp_path)), nprocs=2, join=True,
                       start_method="spawn")
    parts = [np.load(os.path.join(tmp_path, f"r{r}.npz")) for r in range(2)]
    ref = O.netmf_plus(n, s, t, **PRM)
    for p in parts:
        assert p["vol"] == col.size
        assert np.allclose(p["lam"], ref["lam"], rtol=1e-8, atol=1e-10)
        assert np.allclose(p["sigma"], ref["sigma"], rtol=1e-7, atol=1e-9)
    E = np.concatenate([p["E"] for p in parts], axis=0)
    sgn = np.sign((E * ref["E"]).sum(axis=0))
    sgn[sgn == 0] = 1.0
    assert np.abs(E * sgn[None, :] - ref["E"]).max() <= 1e-6 * np.abs(ref["E"]).max()
