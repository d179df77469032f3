#!/usr/bin/env python3
"""Benchmark of the B200-native prlab forward (BASELINE.json metric).

Default workload (N=1, configs[1]): GPT-2 124M, hybrid precision, batch 1,
seq 128, causal -- one "step" is one full forward (embedding -> 12 blocks ->
final LN -> tied LM head, logits [1,128,50257] fp16-lattice) on device.
`--workload c4` runs configs[3] (GPT-2 batch 32, seq 512) instead.
Multi-GPU (torchrun, N>1): every rank runs an independent replica of the same
workload on its own GPU (replicas only: the forward has no exchange step);
value = sequences processed by all ranks / max-over-ranks device time.

Prints ONE JSON line on rank 0.  `--impl reference` times the reference's own
CPU implementation (oracle/_ref/libprlab_ref.so, compiled from the unmodified
reference sources) on the host cores instead.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # name: (preset, batch, seq, policy, description)
    "c2": ("gpt2_small", 1, 128, "hybrid", "C2: GPT-2 124M hybrid FP16, batch 1, seq 128, causal"),
    "c4": ("gpt2_small", 32, 512, "hybrid", "C4: GPT-2 124M hybrid FP16, batch 32, seq 512, causal"),
    "c1": ("bert_base", 1, 128, "hybrid", "BERT-base hybrid FP16, batch 1, seq 128"),
    "c3max": ("bert_base", 32, 512, "hybrid", "BERT-base hybrid FP16, batch 32, seq 512"),
}


def nearest_rank(xs, q):
    """nearest-rank percentile, reference src/bench.cpp:34-45"""
    s = sorted(xs)
    import math
    k = max(1, math.ceil(q * len(s)))
    return s[k - 1]


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return {"hbm_gbs": p["hbm_gbs"], "tflops": p["bf16_tflops"],
                "tflops_sustained": p.get("bf16_tflops_sustained", p["bf16_tflops"]),
                "source": "measured (MEASURED_PEAKS.json)"}
    except Exception:
        return {"hbm_gbs": 6650.0, "tflops": 1590.0, "tflops_sustained": 1400.0,
                "source": "fallback (B200_PROFILING.md)"}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def wait_samples(self, n, timeout=5.0, busy=None):
        """Block (optionally running `busy()` to keep the GPU loaded) until n new samples."""
        start = len(self.lines)
        t0 = time.time()
        while len(self.lines) < start + n and time.time() - t0 < timeout:
            if busy is not None:
                busy()
            else:
                time.sleep(0.01)

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for n, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def model_desc(name):
    import paper_2603_28708_b200 as pg
    return pg.ModelConfig.preset(name)


# ---------------------------------------------------------------------------
# CPU reference (oracle/_ref = the unmodified reference sources, compiled here)
# ---------------------------------------------------------------------------
def cpu_reference_run(cfg, params, S, policy, threads, n_seq, seed):
    """n_seq independent batch-1 sequences over `threads` host threads through
    the reference's prlab::forward; returns (wall seconds, sequences)."""
    from oracle.oracle import ModelConfig as OC, Reference
    ref = Reference()
    oc = OC(**cfg.__dict__)
    import paper_2603_28708_b200 as pg
    ids = pg.random_tokens(cfg.vocab, n_seq, S, seed)
    width = cfg.vocab
    t0 = time.perf_counter()
    ref.forward(oc, params, ids, n_seq, S, policy, threads=threads)
    return time.perf_counter() - t0, n_seq, width


def run_reference_arm(args, wl):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return  # the reference has no multi-GPU path: rank 0 alone runs it
    preset, B, S, policy, desc = WORKLOADS[wl]
    from oracle.oracle import REF_SO
    if not os.path.exists(REF_SO):
        print(json.dumps({"impl": "reference", "unavailable": f"{REF_SO} not built"}))
        return
    import paper_2603_28708_b200 as pg
    cfg = pg.ModelConfig.preset(preset)
    params = pg.build_model(cfg)
    ncores = os.cpu_count() or 1
    threads = max(1, min(ncores, 32))
    # bounded sample: each step runs `threads` batch-1 sequences concurrently
    steps = max(1, min(args.steps, 2))
    warm = 1 if args.warmup > 0 else 0
    for _ in range(warm):
        cpu_reference_run(cfg, params, S, policy, threads, threads, 7)
    walls = []
    for i in range(steps):
        w, n, _ = cpu_reference_run(cfg, params, S, policy, threads, threads, 100 + i)
        walls.append(w)
    total = sum(walls)
    value = steps * threads / total
    line = {
        "impl": "reference",
        "metric": f"sequences/sec ({desc})",
        "value": value, "unit": "seq/s", "n_gpus": args.gpus, "steps": steps, "warmup": warm,
        "ms_per_step": 1000 * total / steps, "p50_latency_ms": 1000 * nearest_rank(walls, 0.5),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32 storage (binary16 emulated)", "data": "synthetic",
        "config": {"workload": desc, "model": preset, "global_batch": B, "seq_len": S,
                   "parallelism": "host threads"},
        "cpu_baseline": {"value": value, "unit": "seq/s", "cores": threads, "kind": "reference",
                         "sample": f"{steps} steps x {threads} concurrent batch-1 seq{S} "
                                   f"{policy} forwards (reference prlab::forward, 1 per thread)"},
        "e2e": {"value": value, "unit": "seq/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def kernel_profile(pg, torch, cfg, B, S, stream, reps=20, causal=1, model=None, d_ids=None, policy="hybrid"):
    """Per-kernel device times of one forward's kernels (inputs resident): each kernel
    replayed `reps` times from a CUDA graph, CUDA events on the stream it runs on.
    With `model` given and a batch-1 shape (forward = the persistent trunk kernel + the
    LM head), the items are exactly those two kernels."""
    M, h, f, V, H, hd = B * S, cfg.hidden, cfg.ffn, cfg.vocab, cfg.heads, cfg.hidden // cfg.heads
    dev = "cuda"
    g = torch.Generator(device=dev).manual_seed(0)
    A = (torch.randn(M, f, device=dev, generator=g) * 0.5).half()
    W = (torch.randn(max(V, f, 3 * h), f, device=dev, generator=g) * 0.02).half()
    bias = torch.zeros(max(V, f, 3 * h), device=dev)
    out16 = torch.empty(M, max((V + 7) // 8 * 8, f, 3 * h), device=dev, dtype=torch.float16)
    out32 = torch.zeros(M, h, device=dev)
    qkv = (torch.randn(M, 3 * h, device=dev, generator=g)).half()
    ctx = torch.empty(M, h, device=dev, dtype=torch.float16)
    L = cfg.num_layers
    ld_head = (V + 7) // 8 * 8
    small = model is not None and model.kernel_count(B, S, policy) == 2
    fl = pg.flop_count(cfg, B, S)
    # trunk: every layer's fp16 weights streamed from HBM once (they exceed L2 across the
    # 12 layers), the embedding rows gathered, the final hidden rows written
    trunk_bytes = L * 2 * (4 * h * h + 2 * h * f) + 2 * 4 * M * h + 2 * M * h
    items = {
        # name: (launch fn, launches per forward, algorithmic bytes, flops)
        "fwd_small": (lambda st: model.forward_trunk_device(d_ids.data_ptr(), B, S, policy, st),
                      1, trunk_bytes, fl["linear"] + fl["attention"]),
        "gemm_qkv": (lambda st: pg.linear_f16_device(A, W, bias, out16, M, 3 * h, h, 3 * h, 0, st),
                     L, 2 * (M * h + 3 * h * h + M * 3 * h), 2 * M * 3 * h * h),
        "gemm_wo": (lambda st: pg.linear_f16_device(A, W, bias, out32, M, h, h, h, 2, st),
                    L, 2 * (M * h + h * h) + 8 * M * h, 2 * M * h * h),
        "gemm_ffn1": (lambda st: pg.linear_f16_device(A, W, bias, out16, M, f, h, f, 1, st),
                      L, 2 * (M * h + h * f + M * f), 2 * M * h * f),
        "gemm_ffn2": (lambda st: pg.linear_f16_device(A, W, bias, out32, M, h, f, h, 2, st),
                      L, 2 * (M * f + h * f) + 8 * M * h, 2 * M * h * f),
        "gemm_head": (lambda st: pg.linear_f16_device(A, W, None, out16, M, V, h, ld_head, 3, st),
                      1, 2 * (M * h + V * h + M * V), 2 * M * h * V),
        "attention": (lambda st: pg.attention_f16_device(qkv, ctx, B, S, H, hd, causal, st),
                      L, 2 * (M * 3 * h + M * h), 4 * B * S * S * h),
    }
    if small:  # the two kernels of the measured step
        items = {k: items[k] for k in ("fwd_small", "gemm_head")}
    else:
        del items["fwd_small"]
    res = {}
    # each kernel is replayed `reps` times from one CUDA graph (as in the forward: PDL-chained,
    # no host launch gaps), timed with CUDA events on the stream the kernels run on
    side = torch.cuda.Stream()
    for name, (fn, count, nbytes, flops) in items.items():
        with torch.cuda.stream(side):
            sp = side.cuda_stream
            for _ in range(3):
                fn(sp)
            side.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=side):
                for _ in range(reps):
                    fn(torch.cuda.current_stream().cuda_stream)
            g.replay()
            side.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(side)
            g.replay()
            e1.record(side)
            side.synchronize()
        t = e0.elapsed_time(e1) / reps / 1000.0
        res[name] = {"us": t * 1e6, "per_forward": count, "bytes": nbytes, "flops": flops,
                     "share_us": t * 1e6 * count}
    return res


def ncu_traffic(wl, kernel):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel` at workload `wl`
    (committed ncu capture summary), or None."""
    path = os.path.join(ROOT, "profiles", "r01", "traffic.json")
    try:
        with open(path) as f:
            t = json.load(f)
        e = t[wl][kernel]
        return {"dram_bytes": float(e["dram_bytes"]), "source": f"profiles/r01/traffic.json ({e['kernel']})"}
    except Exception:
        return None


def run_ours(args, wl):
    import torch
    import paper_2603_28708_b200 as pg

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    preset, B, S, policy, desc = WORKLOADS[wl]
    cfg = pg.ModelConfig.preset(preset)
    params = pg.build_model(cfg)  # reference build_model stream (seed 0)
    model = pg.DeviceModel(cfg, params, device=local)
    V, M = cfg.vocab, B * S
    ld = (V + 7) // 8 * 8
    ids = pg.random_tokens(cfg.vocab, B, S, 1234 + rank)
    d_ids = torch.from_numpy(ids).cuda()
    out16 = torch.empty(M, ld, dtype=torch.float16, device="cuda")
    stream = torch.cuda.current_stream()
    sp = stream.cuda_stream

    def step():
        model.forward_device(d_ids.data_ptr(), B, S, policy, out16.data_ptr(), pg.OUT_F16, ld, sp,
                             True)

    for _ in range(max(3, args.warmup)):
        step()
    model.sync_status(sp)
    kpf = model.kernel_count(B, S, policy)

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- timed region: device-resident inputs; weights (0.25 GB) exceed L2 ----
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]

    def busy():
        for _ in range(8):
            step()
        torch.cuda.synchronize()

    with ClockSampler(local) as clk:
        # the sampler brackets the timed region: >= 2 samples under load before it and
        # one after it (a short timed region can fall between two 100 ms samples)
        clk.wait_samples(2, busy=busy)
        barrier()
        evs[0].record(stream)
        for i in range(args.steps):
            step()
            evs[i + 1].record(stream)
        torch.cuda.synchronize()
        barrier()
        clk.wait_samples(1, busy=busy)
    per_step = [evs[i].elapsed_time(evs[i + 1]) for i in range(args.steps)]
    total_ms = evs[0].elapsed_time(evs[-1])
    model.sync_status(sp)
    if dist is not None:
        t = torch.tensor([total_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    value = world * B * args.steps / (total_ms / 1000.0)

    # ---- e2e: the drop-in C-ABI call with HOST buffers (prlab_gpu_forward) ----
    e2e = None
    if not args.no_e2e:
        h_ids = torch.from_numpy(ids).pin_memory()
        h_logits = torch.empty((B, S, V), dtype=torch.float32).pin_memory()
        ids_np, log_np = h_ids.numpy(), h_logits.numpy()
        for _ in range(max(1, args.warmup)):  # warm the host-path graph and copy-out (W calls)
            _fwd_into(pg, model, ids_np, B, S, policy, log_np)
        e2e_steps = max(3, min(args.steps, 20 if M * V < 50_000_000 else 5))
        barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            _fwd_into(pg, model, ids_np, B, S, policy, log_np)
        t1 = time.perf_counter()
        el = t1 - t0
        if dist is not None:
            t = torch.tensor([el], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            el = float(t.item())
        # under hybrid the library may move the (round16'd) logits as fp16 rows and widen them
        # to fp32 on host threads (host_widen.cpp; chosen by timing on the first call): the
        # PCIe bytes are then half the fp32 result
        widened = model.host_copy_mode(B, S, policy) == 1
        e2e = {"value": world * B * e2e_steps / el, "unit": "seq/s",
               "h2d_bytes_per_step": int(ids_np.nbytes),
               "d2h_bytes_per_step": int(log_np.nbytes // 2 if widened else log_np.nbytes),
               "ms_per_step": 1000 * el / e2e_steps,
               "api": "prlab_gpu_forward (host int32 ids -> host fp32 logits, pinned buffers)"
                      + ("; logits cross PCIe as fp16 rows, widened exactly on host" if widened else "")}

    # ---- roofline of the dominant kernel (standalone CUDA-event timing) ----
    pk = peaks()
    prof = (kernel_profile(pg, torch, cfg, B, S, sp, causal=int(cfg.archetype == 1), model=model,
                           d_ids=d_ids, policy=policy)
            if not args.no_profile else {})
    roof = None
    if prof:
        dom = max(prof, key=lambda k: prof[k]["share_us"])
        d = prof[dom]
        t = d["us"] * 1e-6
        ai = d["flops"] / d["bytes"]
        ridge = pk["tflops"] * 1e12 / (pk["hbm_gbs"] * 1e9)
        if ai < ridge:
            ach = d["bytes"] / t / 1e9
            roof = {"kernel": dom, "bound": "hbm", "achieved": ach, "peak": pk["hbm_gbs"],
                    "unit": "GB/s", "frac": ach / pk["hbm_gbs"], "traffic": None,
                    "algorithmic_bytes": d["bytes"], "launch_us": d["us"]}
        else:
            ach = d["flops"] / t / 1e12
            roof = {"kernel": dom, "bound": "tensor", "achieved": ach, "peak": pk["tflops"],
                    "unit": "TFLOP/s", "frac": ach / pk["tflops"], "traffic": None,
                    "algorithmic_flops": d["flops"], "launch_us": d["us"]}
        roof["peak_source"] = pk["source"]
        # DRAM bytes per launch of the same kernel from one `ncu --set full` capture of this
        # workload (scripts/gpu_ncu_full.sh -> scripts/ncu_traffic.py -> profiles/r01/traffic.json)
        tr = ncu_traffic(wl, dom)
        if tr is not None:
            roof["traffic"] = tr["dram_bytes"]
            roof["traffic_source"] = tr["source"]
            roof["traffic_over_algorithmic"] = tr["dram_bytes"] / d["bytes"]
        roof["breakdown_us_per_forward"] = {k: round(v["share_us"], 2) for k, v in prof.items()}

    # ---- CPU baseline: the reference on this host (rank 0, N=1 only) ----
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            from oracle.oracle import REF_SO
            if os.path.exists(REF_SO):
                threads = max(1, min(os.cpu_count() or 1, 32))
                wall, n, _ = cpu_reference_run(cfg, params, S, policy, threads, threads, 77)
                cpu = {"value": n / wall, "unit": "seq/s", "cores": threads, "kind": "reference",
                       "sample": f"{threads} concurrent batch-1 seq{S} {policy} forwards "
                                 f"(one per thread) through the reference prlab::forward",
                       "latency_ms_per_seq": 1000 * wall}
        except Exception as e:  # reported, never silently replaced
            cpu = {"error": str(e)}

    flops = pg.flop_count(cfg, B, S)["total"]
    line = {
        "metric": f"sequences/sec ({desc})",
        "value": value, "unit": "seq/s", "n_gpus": world, "steps": args.steps,
        "warmup": max(3, args.warmup), "ms_per_step": total_ms / args.steps,
        "p50_latency_ms": nearest_rank(per_step, 0.5), "p95_latency_ms": nearest_rank(per_step, 0.95),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f16 operands / f32 accumulate (hybrid: fp32 LN, softmax, residual)",
        "data": "synthetic: reference build_model(seed 0) weights, random_tokens ids",
        "config": {"workload": desc, "model": preset, "global_batch": world * B, "seq_len": S,
                   "parallelism": f"replicas x{world} (no collective)", "policy": policy,
                   "l2": "working set > L2 (0.25 GB fp16 weights streamed per step)",
                   "graph": "one CUDA graph per forward"},
        "model_tflops_per_s": flops * value / B / 1e12,
        "gpu_launches": kpf * args.steps,
        "kernels_per_step": kpf,
        "clocks": clk.summary(),
        "roofline": roof,
        "cpu_baseline": cpu,
        "e2e": e2e,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def _fwd_into(pg, model, ids_np, B, S, policy, log_np):
    import ctypes as C
    pol = pg.resolve_policy(policy) if isinstance(policy, str) else policy
    pg._check(pg.lib().prlab_gpu_forward(model._h, ids_np.ctypes.data_as(pg._IP), B, S,
                                         C.byref(pol), log_np.ctypes.data_as(pg._FP), None))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="c2")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-profile", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference_arm(args, args.workload)
    else:
        run_ours(args, args.workload)


if __name__ == "__main__":
    main()
