#!/usr/bin/env python
"""Write tests/golden/cfg2_oracle.npz: the fp64 ORACLE's Alg. 5 on BASELINE.json
configs[2] (R-MAT scale 20, edge factor 3; inputs.CONFIGS[2]) at full size and
full parameters.  Calls only `oracle/` (and the seeded input generator of
`paper_2110_12782_b200.inputs`, which holds none of the method's arithmetic);
nothing here comes from the CUDA path.

Stored (all fp64 unless noted; Alg. 5 :310-323, Alg. 4 :293-302):
  lam          all k eigenvalues of Alg. 2 (step 10 order [R3])
  ritz_gap     |lam_k| - |lam_(k+1)| of the Rayleigh-Ritz values (the cut of step 10)
  sigma        all d singular values of Alg. 4 step 8
  rows         a fixed sample of 2048 vertex ids: the 64 highest-degree vertices,
               64 isolated vertices, the rest uniform (seed 0)
  M_rows       Eq. 3's M = F C F^T on rows[:1024] x rows[:256] (basis-free: any
               orthonormal eigenbasis of Alg. 2's output gives the same M)
  Y_rows       Alg. 4 step 3 sketch Y = f(M^') Psi on `rows`
  Z_rows       Alg. 4 step 6 core sketch Z = Pi^T f(M^') Pi on 192 sampled rows (zrows), + Z_fro
  E_rows       the final embedding (after propagation) on `rows`
  E_raw_rows   E = T sqrt(Sigma) before propagation on `rows`
  sens_sigma   conditioning of Alg. 4 at this input: max over 3 draws of
               max_j |sigma_j' - sigma_j| / sigma_1 over the leading sigma
               (>= 1e-2 sigma_1) when Alg. 4 steps 4-8 run on Y + a random
               perturbation of relative Frobenius size 1e-5 (sens_eps)
  (Y_rows, E_rows, E_raw_rows, Z_rows stored as float32: ~1e-7 relative, far
  inside the 1e-4 / 1e-3 tolerances they are compared at.)
Run:  python scripts/oracle_cfg2.py   (~10 min on 8 host cores)
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
from paper_2110_12782_b200 import inputs  # noqa: E402


def main(out=os.path.join(ROOT, "tests", "golden", "cfg2_oracle.npz")):
    w = inputs.CONFIGS[2]
    prm = w.params()
    n, s, t = inputs.make_graph(w.graph)
    T0 = time.time()
    rowptr, col, deg = O.build_csr(n, s, t)
    a = prm["alpha"]
    X = lambda M: O.normalized_spmm(rowptr, col, deg, M, a)
    k, s1, q = prm["k"], prm["s1"], prm["q"]
    # Alg. 2, written out (as oracle.freigs) to also keep the Ritz values past k
    l = k + s1
    Omega = O.gaussian_matrix(n, l, prm["seed"], O.TAG_OMEGA)
    Q, _, _ = O.eig_svd(X(Omega))
    for _ in range(q):
        Q, _, _ = O.eig_svd(X(X(Q)))
    S = Q.T @ X(Q)
    S = 0.5 * (S + S.T)
    lam_all, Uh = O.sym_eig_abs_sorted(S)
    U = (Q @ Uh)[:, :k]
    lam = lam_all[:k]
    del Q
    print(f"freigs {time.time() - T0:.1f}s", flush=True)
    K, F, C = O.factor_pair(U, lam, deg, a, prm["T"])
    del U
    scale = float(col.size) / (prm["b"] * prm["T"])
    d, s2, s3, z, seed, lm = prm["d"], prm["s2"], prm["s3"], prm["z"], prm["seed"], prm["logmode"]
    # Alg. 4, written out (as oracle.single_pass_svd) to keep Y and Z
    rows_psi, sg_psi, p_psi = O.gen_sparse_sign(n, d + s2, z, seed, O.TAG_PSI)
    Y = O.sketch_y(F, C, scale, rows_psi, sg_psi, p_psi, lm)
    Qy = O.orth_range(Y)                     # Alg. 4 step 4 [R10]: 3 of Y's columns are exactly zero
    rows_pi, sg_pi, p_pi = O.gen_sparse_sign(n, d + s3, z, seed, O.TAG_PI)
    Z = O.sketch_z(F, C, scale, rows_pi, sg_pi, p_pi, lm)
    PtQ = O.sparse_sign_apply_T(rows_pi, sg_pi, Qy)
    Sc = O.core_solve(PtQ, Z)
    Uc, sig_all, _ = np.linalg.svd(Sc)
    Ud = Qy @ Uc[:, :d]
    sig = sig_all[:d]
    E_raw = O.embedding_from_svd(Ud, sig)
    print(f"sketch svd {time.time() - T0:.1f}s", flush=True)
    # conditioning of Alg. 4 steps 4-8 at this input (oracle on its own Y, perturbed)
    rng_s = np.random.default_rng(7)
    sens_eps, sens = 1e-5, 0.0
    lead = sig >= 1e-2 * sig[0]
    for _ in range(3):
        Nn = rng_s.standard_normal(Y.shape)
        Nn[:, np.linalg.norm(Y, axis=0) == 0] = 0.0
        Yp = Y + sens_eps * np.linalg.norm(Y) * Nn / np.linalg.norm(Nn)
        Sp = O.core_solve(O.sparse_sign_apply_T(rows_pi, sg_pi, O.orth_range(Yp)), Z)
        sp_ = np.linalg.svd(Sp, compute_uv=False)[:d]
        sens = max(sens, float(np.abs(sp_ - sig)[lead].max() / sig[0]))
    print(f"sensitivity {sens:.3g} at {sens_eps}", flush=True)
    E = O.spectral_propagate(rowptr, col, deg, E_raw, prm["prop_order"], prm["mu"], prm["theta"])
    print(f"propagate {time.time() - T0:.1f}s", flush=True)
    rng = np.random.default_rng(0)
    hubs = np.argsort(-deg, kind="stable")[:64]
    iso = np.flatnonzero(deg == 0)[:64]
    uni = rng.choice(n, 2048 - 128, replace=False)
    rows = np.unique(np.concatenate([hubs, iso, uni])).astype(np.int64)
    M_rows = F[rows[:1024]] @ C @ F[rows[:256]].T
    zrows = np.sort(rng.choice(d + s3, 192, replace=False))
    f32 = lambda a: np.asarray(a, dtype=np.float32)
    np.savez_compressed(
        out, n=n, k=k, d=d, h2=d + s2, h3=d + s3, lam=lam, lam_all=lam_all, ritz_gap=abs(lam_all[k - 1]) - abs(lam_all[k]),
        sigma=sig, sigma_all=sig_all, rows=rows, M_rows=M_rows, sens_sigma=sens, sens_eps=sens_eps, Y_rows=f32(Y[rows]), Y_fro=np.linalg.norm(Y),
        zrows=zrows, Z_rows=f32(Z[zrows]), Z_fro=np.linalg.norm(Z), E_rows=f32(E[rows]), E_raw_rows=f32(E_raw[rows]),
        E_col_norms=np.linalg.norm(E, axis=0), E_raw_col_norms=np.linalg.norm(E_raw, axis=0),
        rank_Y=Qy.shape[1], zero_cols_Y=np.flatnonzero(np.linalg.norm(Y, axis=0) == 0),
        wall_s=time.time() - T0)
    print(f"wrote {out} in {time.time() - T0:.1f}s; lam[:4]={lam[:4]} sigma[:4]={sig[:4]}")


if __name__ == "__main__":
    main(*sys.argv[1:])
