"""LM-head tile choice at M = 256 (C3 batch 2 x 128 / 4 x 64 / 8 x 32): 1-CTA vs CTA-pair
kernel and BN, EPI_F16, CUDA-graph replay of 20 back-to-back launches (L2-warm weights)."""
import json, os, sys
sys.path.insert(0, os.path.join(os.environ.get("GRAFT_REPO_ROOT", "."), "scripts"))
from sweep_gemm import time_cfg
for (M, N) in [(256, 30522), (256, 50257), (128, 30522)]:
    for bn in (0, 256, 128, 64):
        for ln in (0, 1, 2):
            try:
                us, tf, gbs = time_cfg(M, N, 768, 3, bn, 1, ln)
                print(json.dumps({"M": M, "N": N, "bn": bn, "lean": ln, "us": round(us, 2), "gbs": round(gbs, 1)}), flush=True)
            except Exception as e:
                print(json.dumps({"M": M, "N": N, "bn": bn, "lean": ln, "err": str(e)[:100]}))
