#!/usr/bin/env python3
"""Memory planner evidence (north_star subsystem 1): device bytes of the
hybrid plan vs an all-fp32 plan at C4 (GPT-2, batch 32, seq 512) and C3-max (BERT 32x512),
from the library's own accounting (prlab_gpu_model_memory_ex) and from cudaMemGetInfo
deltas around model creation and the first forward of each policy.  One JSON line per
model.  The fp32 plan runs the generic path (fp32 weights materialised, fp32 activations)."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2603_28708_b200 as pg  # noqa: E402


def used():
    torch.cuda.synchronize()
    free, total = torch.cuda.mem_get_info()
    return total - free


def run(name, B, S):
    cfg = pg.ModelConfig.preset(name)
    params = pg.build_model(cfg)
    ids = torch.from_numpy(pg.random_tokens(cfg.vocab, B, S, 1)).cuda()
    st = torch.cuda.current_stream().cuda_stream
    out = {"model": name, "batch": B, "seq": S, "param_count": int(params.size),
           "reference_fp32_param_bytes": int(params.size) * 4}
    for pol in ("hybrid", "fp32"):
        u0 = used()
        m = pg.DeviceModel(cfg, params)
        u1 = used()
        if pol == "hybrid":
            # the C4 replica step: forward + fused NLL head (no [B*S, V] logits in the library)
            tg = torch.roll(ids, -1)
            nll = torch.empty(B * S, dtype=torch.float64, device="cuda")
            m.forward_nll_device(ids.data_ptr(), tg.data_ptr(), B, S, pol, nll.data_ptr(), 0, st)
        else:
            lg = torch.empty(B * S, cfg.vocab, dtype=torch.float32, device="cuda")
            m.forward_device(ids.data_ptr(), B, S, pol, lg.data_ptr(), pg.OUT_F32, cfg.vocab, st, False)
            del lg
        m.sync_status(st)
        u2 = used()
        rep = m.memory_report()
        out[pol] = {"library": rep, "device_delta_create": u1 - u0,
                    "device_delta_after_forward": u2 - u0}
        m.close()
        del m
        torch.cuda.synchronize()
    h, f = out["hybrid"]["library"], out["fp32"]["library"]
    # an all-fp32 model holds every parameter in fp32 (what the reference keeps resident)
    out["weights_hybrid_over_all_fp32"] = h["weights_fast"] / out["reference_fp32_param_bytes"]
    out["activations_hybrid_over_fp32_plan"] = (h["workspace"] + h["logits"]) / (f["workspace"] + f["logits"])
    out["resident_hybrid_over_fp32_plan"] = h["total"] / (out["reference_fp32_param_bytes"] + f["workspace"]
                                                          + f["logits"] + f["scratch"])
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    run("gpt2_small", 32, 512)
    run("bert_base", 32, 512)
