#!/usr/bin/env python3
"""C3: BERT-base hybrid sweep, batch {1,2,4,8,16,32} x seq {32,64,128,256,512} on one B200.
Per config: p50 / p95 device latency of one forward (CUDA-graph replay, 20 steps, CUDA
events), sequences/s, and fidelity of every logit against the GPU fp32 forward (the fp32
SIMT path is pinned to the CPU reference within 1e-3 relative in tests/test_gpu_forward.py):
cosine, max |diff|, non-finite count.  One JSON line per config."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2603_28708_b200 as pg  # noqa: E402


def nearest_rank(xs, q):
    s = sorted(xs)
    return s[max(1, int(np.ceil(q * len(s)))) - 1]


def main():
    cfg = pg.ModelConfig.preset("bert_base")
    model = pg.DeviceModel(cfg, pg.build_model(cfg))
    V = cfg.vocab
    st = torch.cuda.current_stream()
    for B in (1, 2, 4, 8, 16, 32):
        for S in (32, 64, 128, 256, 512):
            ids = torch.from_numpy(pg.random_tokens(V, B, S, 7 * B + S)).cuda()
            out = torch.empty(B * S, V, device="cuda", dtype=torch.float32)
            for _ in range(3):
                model.forward_device(ids.data_ptr(), B, S, "hybrid", out.data_ptr(), pg.OUT_F32, V, st.cuda_stream, True)
            torch.cuda.synchronize()
            evs = [torch.cuda.Event(enable_timing=True) for _ in range(21)]
            evs[0].record(st)
            for i in range(20):
                model.forward_device(ids.data_ptr(), B, S, "hybrid", out.data_ptr(), pg.OUT_F32, V, st.cuda_stream, True)
                evs[i + 1].record(st)
            torch.cuda.synchronize()
            ms = [evs[i].elapsed_time(evs[i + 1]) for i in range(20)]
            ref = torch.empty_like(out)
            model.forward_device(ids.data_ptr(), B, S, "fp32", ref.data_ptr(), pg.OUT_F32, V, st.cuda_stream, False)
            model.sync_status(st.cuda_stream)
            cmp = pg.compare_logits_device(ref, out, B * S, V)
            line = {"B": B, "S": S, "p50_ms": round(nearest_rank(ms, 0.5), 4), "p95_ms": round(nearest_rank(ms, 0.95), 4),
                    "seq_per_s": round(B / (np.mean(ms) / 1000), 1), "cosine_vs_fp32": cmp["cosine"],
                    "max_abs_vs_fp32": cmp["max_abs_error"], "nonfinite": cmp["candidate_nonfinite"]}
            print(json.dumps(line), flush=True)
            del out, ref
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
