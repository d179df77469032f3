#!/usr/bin/env python3
"""Device->host copy-out of batch-1 logits (GPT-2: 128 x 50257 fp16, device pitch padded to
8 elements): PCIe rate of 2D (pitched) vs 1D (dense) copies, chunked vs single, and of SM
stores into mapped pinned memory (zero-copy).  One JSON line per variant."""
import ctypes as C
import json
import time

import torch

rt = C.CDLL("libcudart.so.12")
rows, cols = 128, 50257
ld = (cols + 7) // 8 * 8
dev = torch.randn(rows, ld, device="cuda").half()
dense = torch.empty(rows * cols, device="cuda", dtype=torch.float16)
host = torch.empty(rows * cols, dtype=torch.float16, pin_memory=True)
st = torch.cuda.current_stream()
s = C.c_void_p(st.cuda_stream)
D2H = 2


def timed(fn, n=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
        torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e6


def cp2d(chunks):
    per = (rows + chunks - 1) // chunks

    def f():
        for c in range(0, rows, per):
            nr = min(per, rows - c)
            rt.cudaMemcpy2DAsync(C.c_void_p(host.data_ptr() + c * cols * 2), C.c_size_t(cols * 2),
                                 C.c_void_p(dev.data_ptr() + c * ld * 2), C.c_size_t(ld * 2),
                                 C.c_size_t(cols * 2), C.c_size_t(nr), D2H, s)
    return f


def cp1d(chunks, compact):
    n = rows * cols * 2
    per = (n + chunks - 1) // chunks

    def f():
        if compact:
            dense.view(rows, cols).copy_(dev[:, :cols])
        for o in range(0, n, per):
            rt.cudaMemcpyAsync(C.c_void_p(host.data_ptr() + o), C.c_void_p(dense.data_ptr() + o),
                               C.c_size_t(min(per, n - o)), D2H, s)
    return f


nbytes = rows * cols * 2
for name, fn in [("2d_x1", cp2d(1)), ("2d_x16", cp2d(16)), ("1d_x1", cp1d(1, False)), ("1d_x16", cp1d(16, False)),
                 ("compact+1d_x1", cp1d(1, True)), ("compact+1d_x16", cp1d(16, True)), ("compact_only", lambda: dense.view(rows, cols).copy_(dev[:, :cols]))]:
    us = timed(fn)
    print(json.dumps({"variant": name, "us": round(us, 1), "GB/s": round(nbytes / us / 1e3, 1)}))
# zero-copy: device kernel (torch copy) writing into the mapped pinned buffer
hv = host.view(rows, cols)
# torch cannot target host memory from a kernel; use cudaHostGetDevicePointer + a 1D device copy kernel via cudaMemcpyAsync D2D
dptr = C.c_void_p()
rt.cudaHostGetDevicePointer(C.byref(dptr), C.c_void_p(host.data_ptr()), 0)
print(json.dumps({"mapped_devptr_ok": bool(dptr.value)}))
if dptr.value:
    def zc():
        rt.cudaMemcpyAsync(dptr, C.c_void_p(dense.data_ptr()), C.c_size_t(nbytes), 3, s)  # D2D into mapped host
    us = timed(zc)
    print(json.dumps({"variant": "d2d_into_mapped_host", "us": round(us, 1), "GB/s": round(nbytes / us / 1e3, 1)}))


# chunks spread round-robin over several copy streams (per-copy setup overlaps)
def cp2d_multi(chunks, nstreams):
    per = (rows + chunks - 1) // chunks
    streams = [torch.cuda.Stream() for _ in range(nstreams)]
    evs = [torch.cuda.Event() for _ in range(chunks)]
    start = torch.cuda.Event()

    def f():
        start.record(st)
        for i, c in enumerate(range(0, rows, per)):
            ss = streams[i % nstreams]
            ss.wait_event(start)
            nr = min(per, rows - c)
            rt.cudaMemcpy2DAsync(C.c_void_p(host.data_ptr() + c * cols * 2), C.c_size_t(cols * 2),
                                 C.c_void_p(dev.data_ptr() + c * ld * 2), C.c_size_t(ld * 2),
                                 C.c_size_t(cols * 2), C.c_size_t(nr), D2H, C.c_void_p(ss.cuda_stream))
            evs[i].record(ss)
        for e in evs:
            e.synchronize()
    return f


for ch, ns in [(16, 2), (16, 4), (8, 2), (8, 1), (4, 1), (4, 2)]:
    us = timed(cp2d_multi(ch, ns))
    print(json.dumps({"variant": f"2d_x{ch}_streams{ns}", "us": round(us, 1), "GB/s": round(nbytes / us / 1e3, 1)}))
