"""Dump the compacted (isolated vertices dropped, original order) CSR of a
BASELINE config for scripts/dbg/spmm_lab.cu: int64 n, nnz, rowptr[n+1], int32 col."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_2110_12782_b200 import inputs
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
out = sys.argv[2] if len(sys.argv) > 2 else "/tmp/csr.bin"
n, s, t = inputs.make_graph(inputs.CONFIGS[cfg].graph)
s = s.astype(np.int64); t = t.astype(np.int64)
k = s != t
u = np.concatenate([s[k], t[k]]); v = np.concatenate([t[k], s[k]])
key = np.unique(u * n + v)
u, v = key // n, key % n
deg = np.bincount(u, minlength=n)
keep = deg > 0
m = np.cumsum(keep) - 1
u, v = m[u], m[v]
nc = int(keep.sum())
rp = np.zeros(nc + 1, np.int64)
np.cumsum(np.bincount(u, minlength=nc), out=rp[1:])
with open(out, "wb") as f:
    np.array([nc, v.size], np.int64).tofile(f)
    rp.tofile(f)
    v.astype(np.int32).tofile(f)
print("wrote", out, nc, v.size)
