import sys, os, numpy as np
sys.path.insert(0, '/root/repo') if os.path.exists('/root/repo') else None
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import paper_2603_28708_b200 as pg
from oracle.oracle import Oracle, ModelConfig as OC, compare_logits
cfg = pg.ModelConfig.preset("gpt2_small")
params = pg.build_model(cfg)
m = pg.DeviceModel(cfg, params)
for B, S in [(1, 128), (1, 37), (2, 64)]:
    ids = pg.random_tokens(cfg.vocab, B, S, 7)
    got = m.forward(ids, B, S, "hybrid")
    os.environ["PRLAB_NO_FWD_SMALL"] = "1"
    m2 = pg.DeviceModel(cfg, params)
    ref = m2.forward(ids, B, S, "hybrid")
    del os.environ["PRLAB_NO_FWD_SMALL"]
    m2.close()
    r = compare_logits(ref, got)
    print(B, S, "vs multi-kernel fast path:", r["cosine"], r["max_abs_error"], r["candidate_nonfinite"], flush=True)
