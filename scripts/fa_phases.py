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
    dbg = torch.zeros(256 + 2 * 1024, dtype=torch.int64, device="cuda")
    pg._check(pg.lib().prlab_gpu_attention_f16_device_dbg(C.c_void_p(qkv.data_ptr()), C.c_void_p(ctx.data_ptr()),
                                                          B, S, H, hd, 1, None, C.c_void_p(dbg.data_ptr())))
    torch.cuda.synchronize()
    raw = dbg.cpu().numpy().astype(np.float64)
    d = raw[:256].reshape(32, 8)
    sp = raw[256:].reshape(-1, 2)
    sp = sp[sp[:, 0] > 0]
    if len(sp):
        t0 = sp[:, 0].min()
        st, en = (sp[:, 0] - t0) / 1e3, (sp[:, 1] - t0) / 1e3
        print(json.dumps({"ctas": len(sp), "start_us_max": round(float(st.max()), 2),
                          "end_us": {"min": round(float(en.min()), 2), "median": round(float(np.median(en)), 2),
                                     "p90": round(float(np.percentile(en, 90)), 2), "max": round(float(en.max()), 2)},
                          "cta0_end_us": round(float(en[0]), 2)}))
        # static schedule (attn_fa.cu fa_unit_at / fa_decode): blocks and units per CTA vs end time
        g, items, nqt = len(sp), B * H, (S + 127) // 128
        n = items * nqt
        loads = []
        for c in range(g):
            blocks = units = 0
            for k in range(64):
                u = k * g + ((g - 1 - c) if (k & 1) else c)
                if u >= n:
                    break
                qt = nqt - 1 - u // items
                blocks += qt + 1
                units += 1
            loads.append((blocks, units))
        by = {}
        for c in range(g):
            by.setdefault(loads[c], []).append(en[c])
        print(json.dumps({"end_us_by_blocks_units": {f"{k[0]}b/{k[1]}u": round(float(np.mean(v)), 2) for k, v in sorted(by.items())},
                          "sm_pair_end_us": [round(float(max(en[c], en[c + g // 2])), 1) for c in range(0, g // 2, 16)],
                          "end_first_half_vs_second": [round(float(np.mean(en[:g // 2])), 2), round(float(np.mean(en[g // 2:])), 2)]}))
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
