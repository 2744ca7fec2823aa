"""Dump the CUDA path's configs[2] outputs (lambda, sigma, sketch samples,
Eq. 3 samples) for offline analysis against tests/golden/cfg2_oracle.npz."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import test_gpu_cfg2 as T
rows = np.load(T.GOLD)["rows"]
out = T.run_cfg2(rows, extra=True)
flat = {}
for k, v in out.items():
    if isinstance(v, dict):
        for k2, v2 in v.items():
            flat[f"{k}_{k2}"] = v2
    else:
        flat[k] = v
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
np.savez_compressed(os.path.join(ROOT, "gpurun_out", "cfg2_gpu.npz"), **flat)
print("ok", sorted(flat))
