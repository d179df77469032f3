"""N-tile rule check for the 1-CTA / pair tcgen05 GEMM across the forward's shapes:
auto (plan_gemm_tc's choice) vs forced BN 256 / 128 / 64, EPI_F16, L2-warm graph replay."""
import json, os, sys
sys.path.insert(0, os.path.join(os.environ.get("GRAFT_REPO_ROOT", "."), "scripts"))
from sweep_gemm import time_cfg
for M in (128, 256, 512, 1024, 2048, 4096):
    for (N, K) in [(2304, 768), (768, 768), (3072, 768), (768, 3072), (30522, 768), (50257, 768)]:
        r = {"M": M, "N": N, "K": K}
        for bn in (0, 256, 128, 64):
            try:
                us, tf, gbs = time_cfg(M, N, K, 3, bn, 0, 0)
                r[str(bn)] = round(us, 2)
            except Exception as e:
                r[str(bn)] = str(e)[:60]
        print(json.dumps(r), flush=True)
