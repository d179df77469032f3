#!/usr/bin/env python3
"""Per-block phase timeline of the streaming attention kernel (attn_fa.cu), CTA 0, clock64:
softmax warp: S ready seen -> pass 1 done -> max barrier -> P ready (arrive); MMA thread:
P ready seen -> P.V + next Q.K^T issued; plus the gaps between them.  C4 shape by default."""
import ctypes as C
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_28708_b200 as pg  # noqa: E402


def main():
    B, S, H, hd = int(os.environ.get("B", 32)), int(os.environ.get("S", 512)), 12, 64
    qkv = (torch.randn(B * S, 3 * H * hd, device="cuda") * 1.5).half()
    ctx = torch.empty(B * S, H * hd, device="cuda", dtype=torch.float16)
    for _ in range(3):
        pg.attention_f16_device(qkv, ctx, B, S, H, hd, 1)
    dbg = torch.zeros(32 * 8, dtype=torch.int64, device="cuda")
    pg._check(pg.lib().prlab_gpu_attention_f16_device_dbg(C.c_void_p(qkv.data_ptr()), C.c_void_p(ctx.data_ptr()),
                                                          B, S, H, hd, 1, None, C.c_void_p(dbg.data_ptr())))
    torch.cuda.synchronize()
    d = dbg.cpu().numpy().reshape(32, 8).astype(np.float64)
    rows = []
    for b in range(1, 31):
        if d[b, 0] == 0 or d[b + 1, 0] == 0:
            break
        rows.append({"pass1": d[b, 1] - d[b, 0], "max_bar": d[b, 2] - d[b, 1], "pass2_to_ready": d[b, 3] - d[b, 2],
                     "ready_to_mma_seen": d[b, 4] - d[b, 3], "mma_issue": d[b, 5] - d[b, 4],
                     "issue_to_next_s_seen": d[b + 1, 0] - d[b, 5], "block_total": d[b + 1, 0] - d[b, 0],
                     # row-owner kernel: first chunk loaded, all chunks packed (0 / unused otherwise)
                     "row_first_chunk": d[b, 6] - d[b, 0] if d[b, 6] else 0,
                     "row_all_chunks": d[b, 7] - d[b, 0] if d[b, 7] else 0})
    avg = {k: round(float(np.median([r[k] for r in rows])), 1) for k in rows[0]}
    n = int((d[:, 0] > 0).sum())
    print(json.dumps({"cta0_blocks": n, "s_seen_deltas": [int(d[i + 1, 0] - d[i, 0]) for i in range(n - 1)],
                      "span_cycles": int(d[n - 1, 3] - d[0, 0])}))
    print(json.dumps({"B": B, "S": S, "blocks": len(rows), "median_cycles": avg}))


if __name__ == "__main__":
    main()
