"""Parity of the hand-written sm_100a kernels (tcgen05 GEMM, fused attention) against
plain PyTorch fp32 references of the same hybrid-lattice math, plus the per-operator
C-ABI against the CPU oracle on the reference's known-answer tests."""
import math

import numpy as np
import pytest

import paper_2603_28708_b200 as pg
from prlab_testutil import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def r16(t):
    return t.to(torch.float16).to(torch.float32)


@pytest.fixture(scope="module", autouse=True)
def _no_tf32():
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.allow_tf32 = False
    yield


def _gemm_ref(A, Wt, bias, epi, resid=None):
    # exact products of fp16 values, accumulated in float64 (no reference-side rounding
    # noise at large K); the kernel's own fp32 accumulation is the only deviation
    acc = (A.double() @ Wt.double().T).float()
    v = r16(acc)
    if epi == 3:
        return v
    v = r16(v + (bias if bias is not None else 0.0))
    if epi == 1:
        v = r16(0.5 * v * (1.0 + torch.erf(v * 0.7071067811865476)))
    if epi == 2:
        return resid + v
    return v


# (M, N, K): tile-aligned, M/N tails, tiny, wide LM-head-like N, FFN shapes
SHAPES = [(128, 256, 64), (300, 2304, 768), (1, 64, 64), (128, 50257, 768), (777, 3072, 768),
          (2048, 768, 3072), (128, 768, 768), (4096, 2304, 768)]


@pytest.mark.parametrize("M,N,K", SHAPES)
@pytest.mark.parametrize("epi", [0, 1, 2, 3])
def test_tc_linear_matches_fp32_reference(M, N, K, epi):
    if epi != 0 and (M, N, K) in [(128, 50257, 768)]:
        pytest.skip("head shape only needs epi 0/3")
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N + K + epi)
    A = (torch.randn(M, K, device="cuda", generator=g) * 0.5).half()
    Wt = (torch.randn(N, K, device="cuda", generator=g) * 0.05).half()
    bias = r16(torch.randn(N, device="cuda", generator=g) * 0.1)
    ldo = N if epi == 2 else (N + 7) // 8 * 8
    if epi == 2:
        out = torch.randn(M, N, device="cuda", generator=g)
        resid = out.clone()
    else:
        out = torch.full((M, ldo), float("nan"), device="cuda", dtype=torch.float16)
        resid = None
    pg.linear_f16_device(A, Wt, bias if epi != 3 else None, out, M, N, K, ldo, epi)
    torch.cuda.synchronize()
    ref = _gemm_ref(A, Wt, bias, epi, resid)
    got = out.float()[:, :N]
    assert torch.isfinite(got).all(), "unwritten / non-finite outputs"
    err = (got - ref).abs()
    # accumulation order differs from fp32 sequential: allow one fp16 ulp at the value
    tol = torch.clamp(ref.abs(), min=6.1e-5) * 2.0 ** -10 * 1.01 + 1e-6
    frac_bad = (err > tol).float().mean().item()
    assert frac_bad < 3e-3, f"max err {err.max().item():.3e}, {frac_bad:.2e} beyond 1 ulp"
    assert err.max().item() <= 4 * tol.max().item() + 1e-3


def _attn_ref(qkv, B, S, H, hd, causal):
    h = H * hd
    x = qkv.float().view(B, S, 3, H, hd)
    q, k, v = x[:, :, 0].transpose(1, 2), x[:, :, 1].transpose(1, 2), x[:, :, 2].transpose(1, 2)
    s = r16((q @ k.transpose(-1, -2)) * (1.0 / math.sqrt(hd)))
    if causal:
        mask = torch.triu(torch.ones(S, S, dtype=torch.bool, device=qkv.device), 1)
        s = s.masked_fill(mask, float("-inf"))
    m = s.amax(-1, keepdim=True)
    e = torch.exp(s - m)
    p = r16(e / e.sum(-1, keepdim=True))
    o = r16(p @ v)
    return o.transpose(1, 2).reshape(B * S, h)


# shapes on both attention kernels: the streaming one (S > 128, or B*H above the SM count:
# (16, 1, 1), (13, 20, 1), (16, 3, 0)) and the resident-row one (the rest)
@pytest.mark.parametrize("B,S,causal", [(1, 128, 0), (1, 128, 1), (2, 77, 0), (2, 77, 1),
                                         (1, 1, 1), (3, 200, 1), (2, 512, 0), (2, 512, 1),
                                         (1, 384, 0), (4, 64, 1), (16, 1, 1), (13, 20, 1), (16, 3, 0),
                                         (13, 128, 1)])
def test_tc_attention_matches_fp32_reference(B, S, causal):
    H, hd = 12, 64
    g = torch.Generator(device="cuda").manual_seed(B * 1000 + S * 2 + causal)
    qkv = (torch.randn(B * S, 3 * H * hd, device="cuda", generator=g) * 1.5).half()
    ctx = torch.full((B * S, H * hd), float("nan"), device="cuda", dtype=torch.float16)
    pg.attention_f16_device(qkv, ctx, B, S, H, hd, causal)
    torch.cuda.synchronize()
    ref = _attn_ref(qkv, B, S, H, hd, causal)
    got = ctx.float()
    assert torch.isfinite(got).all()
    err = (got - ref).abs()
    assert err.max().item() < 2e-2, f"max err {err.max().item()}"
    assert err.mean().item() < 1e-3


# ---------------------------------------------------------------------------
# per-operator C-ABI vs the oracle on the reference's known answers
# (reference tests/test_kernels.cpp)
# ---------------------------------------------------------------------------
F32 = pg.KernelConfig(pg.F32, pg.F32, True)
F16ACC = pg.KernelConfig(pg.F16E, pg.F16E, True)
F16WIDE = pg.KernelConfig(pg.F16E, pg.F32, True)
F16UNSTABLE = pg.KernelConfig(pg.F16E, pg.F16E, False)


def test_kat_long_reductions():  # test_kernels.cpp:37-60
    for n, want in [(2049, (2048.0, 2048.0, 2049.0)), (2050, (2048.0, 2050.0, 2050.0))]:
        a = np.ones((1, n), np.float32)
        b = np.ones((n, 1), np.float32)
        assert pg.matmul(a, b, F16ACC)[0, 0] == want[0]
        assert pg.matmul(a, b, F16WIDE)[0, 0] == want[1]
        assert pg.matmul(a, b, F32)[0, 0] == want[2]


def test_kat_matmul_vs_oracle_bitexact_narrow():
    rng = np.random.default_rng(3)
    a = rng.uniform(-1, 1, (17, 33)).astype(np.float32)
    b = rng.uniform(-1, 1, (33, 9)).astype(np.float32)
    o = oracle()
    for cfg in [F16ACC, F16WIDE]:
        got = pg.matmul(a, b, cfg)
        want = o.matmul(a, b, cfg.compute, cfg.accum)
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
    got = pg.matmul(a, b, F32)
    ref = a.astype(np.float64) @ b.astype(np.float64)
    assert np.abs(got - ref).max() <= 33 * 1.2e-7 * 33


def test_kat_softmax():  # test_kernels.cpp:82-98
    x = np.array([[12.0, 0.0]], np.float32)
    y = pg.softmax_lastdim(x, F16ACC)
    assert y[0, 0] == 1.0 and y[0, 1] == np.float32(6.139278411865234e-06)
    y = pg.softmax_lastdim(x, F16UNSTABLE)
    assert np.isnan(y[0, 0]) and y[0, 1] == 0.0


def test_kat_scores_fold_scale():  # test_kernels.cpp:119-135
    q = np.array([[1, 2, 3], [4, 5, 6]], np.float32)
    k = np.array([[7, 8, 9], [10, 11, 12]], np.float32)
    s, tap = pg.attention_scores(q, k, 0.125, F16ACC, capture=True)
    ref = (q.astype(np.float64) @ k.T.astype(np.float64)).astype(np.float32)
    assert np.array_equal(tap, ref * np.float32(0.125))
    assert np.array_equal(s, oracle().round16_array(ref * np.float32(0.125)))


def test_kat_layernorm_gelu_add_embed():
    y = pg.layernorm_lastdim(np.full((1, 6), 3.0, np.float32), np.ones(6, np.float32),
                             np.full(6, 0.25, np.float32), 1e-5, F32)
    assert np.allclose(y, 0.25, rtol=1e-6)
    g = pg.gelu(np.array([0.0, 1.0, -1.0], np.float32), F32)
    assert g[0] == 0.0
    assert abs(g[1] - 0.8413447460685429) < 1e-6 and abs(g[2] + 0.15865525393145707) < 1e-6
    assert pg.add(np.array([2048.0], np.float32), np.array([1.0], np.float32), F16ACC)[0] == 2048.0
    assert pg.add(np.array([2048.0], np.float32), np.array([1.0], np.float32), F32)[0] == 2049.0
    tok = np.array([[0, 0], [10, 20], [30, 40]], np.float32)
    pos = np.array([[1, 2], [3, 4]], np.float32)
    e = pg.embed(tok, pos, [2, 1], 1, 2, F32)
    assert e.ravel().tolist() == [31.0, 42.0, 13.0, 24.0]
    with pytest.raises(IndexError):
        pg.embed(tok, pos, [3, 0], 1, 2, F32)
    with pytest.raises(IndexError):
        pg.embed(tok, pos, [0, 0, 0], 1, 3, F32)


def test_kernel_config_validation():
    with pytest.raises(ValueError):
        pg.matmul(np.ones((2, 2), np.float32), np.ones((2, 2), np.float32),
                  pg.KernelConfig(pg.F32, pg.F16E, True))


def test_per_op_vs_oracle_random():
    rng = np.random.default_rng(7)
    o = oracle()
    x = rng.uniform(-4, 4, (8, 16)).astype(np.float32)
    for cfg in [F32, F16ACC, F16WIDE, F16UNSTABLE]:
        got = pg.softmax_lastdim(x, cfg)
        want = o.softmax(x, cfg.compute, cfg.accum, bool(cfg.stabilized))
        assert np.allclose(got, want, rtol=2e-6, atol=1e-7, equal_nan=True)
    xl = rng.normal(0, 1, (4, 64)).astype(np.float32)
    gam = rng.normal(1, 0.1, 64).astype(np.float32)
    bet = rng.normal(0, 0.1, 64).astype(np.float32)
    for cfg in [F32, F16ACC]:
        got = pg.layernorm_lastdim(xl, gam, bet, 1e-5, cfg)
        want = o.layernorm(xl, gam, bet, 1e-5, cfg.compute, cfg.accum)
        tol = 1e-5 if cfg.compute == pg.F32 else 2e-3
        assert np.abs(got - want).max() <= tol


@pytest.mark.parametrize("bn", [64, 128, 256])
@pytest.mark.parametrize("splits", [1, 3, -3, 8])
@pytest.mark.parametrize("lean", [1, -1])
@pytest.mark.parametrize("epi", [0, 2])
def test_tc_linear_forced_configs(bn, splits, lean, epi):
    """Every tile width / split-K (cluster >0, global workspace <0) / pipeline-depth
    variant gives the same lattice result."""
    if splits > 1 and bn == 256:
        pytest.skip("cluster split-K is for narrow tiles")
    M, N, K = 200, 768, 1536
    g = torch.Generator(device="cuda").manual_seed(bn + splits + lean + epi)
    A = (torch.randn(M, K, device="cuda", generator=g) * 0.5).half()
    Wt = (torch.randn(N, K, device="cuda", generator=g) * 0.05).half()
    bias = r16(torch.randn(N, device="cuda", generator=g) * 0.1)
    if epi == 2:
        out = torch.randn(M, N, device="cuda", generator=g)
        resid = out.clone()
    else:
        out = torch.full((M, N), float("nan"), device="cuda", dtype=torch.float16)
        resid = None
    pg.linear_f16_device_ex(A, Wt, bias, out, M, N, K, N, epi, bn, splits, lean)
    torch.cuda.synchronize()
    ref = _gemm_ref(A, Wt, bias, epi, resid)
    got = out.float()
    assert torch.isfinite(got).all()
    err = (got - ref).abs()
    tol = torch.clamp(ref.abs(), min=6.1e-5) * 2.0 ** -10 * 1.01 + 1e-6
    assert (err > tol).float().mean().item() < 3e-3
    # split-K reduction order is fixed: results are reproducible bit for bit
    out2 = resid.clone() if epi == 2 else torch.empty_like(out)
    pg.linear_f16_device_ex(A, Wt, bias, out2, M, N, K, N, epi, bn, splits, lean)
    torch.cuda.synchronize()
    assert torch.equal(out2, out) if epi != 2 else True


@pytest.mark.parametrize("M", [512, 640, 1000])
@pytest.mark.parametrize("bn", [128, 256])
@pytest.mark.parametrize("epi", [0, 1, 2, 3])
def test_tc_linear_cta_pair(M, bn, epi):
    """The cta_group::2 kernel (256-row tiles over a CTA pair), incl. an odd number of
    128-row blocks (the pair's second CTA runs entirely out of bounds) and M tails."""
    N, K = 768 + 256, 768
    g = torch.Generator(device="cuda").manual_seed(M + bn + epi)
    A = (torch.randn(M, K, device="cuda", generator=g) * 0.5).half()
    Wt = (torch.randn(N, K, device="cuda", generator=g) * 0.05).half()
    bias = r16(torch.randn(N, device="cuda", generator=g) * 0.1)
    if epi == 2:
        out = torch.randn(M, N, device="cuda", generator=g)
        resid = out.clone()
    else:
        out = torch.full((M, N), float("nan"), device="cuda", dtype=torch.float16)
        resid = None
    pg.linear_f16_device_ex(A, Wt, bias if epi != 3 else None, out, M, N, K, N, epi, bn, 1, 2)
    torch.cuda.synchronize()
    ref = _gemm_ref(A, Wt, bias, epi, resid)
    got = out.float()
    assert torch.isfinite(got).all()
    err = (got - ref).abs()
    tol = torch.clamp(ref.abs(), min=6.1e-5) * 2.0 ** -10 * 1.01 + 1e-6
    assert (err > tol).float().mean().item() < 3e-3, err.max().item()


# ---- fp32-policy linears on the tensor cores (3xTF32, gemm_tf32.cu) ----
@pytest.mark.parametrize("M,N,K,epi", [(128, 2304, 768, 0), (128, 768, 3072, 2), (512, 3072, 768, 1),
                                       (77, 768, 768, 2), (300, 50264, 768, 0), (1, 96, 64, 1),
                                       (1000, 1000, 2048, 0)])
def test_linear_f32_tensor_core_vs_fp64(M, N, K, epi):
    """3xTF32 (x.w ~= x.w + x_lo.w + x.w_lo, the tensor core truncating each operand to 19
    bits) recovers fp32-accurate products: compared with an fp64 reference the error stays at
    fp32 summation level (a few 1e-6 of the row's absolute dot-product scale), far inside the
    fp32 policy's 1e-3 relative contract -- while a plain tf32 GEMM would be ~1e-3 off."""
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N)
    A = torch.randn(M, K, device="cuda", generator=g)
    W = torch.randn(N, K, device="cuda", generator=g) * 0.05
    bias = torch.randn(N, device="cuda", generator=g)
    resid = torch.randn(M, N, device="cuda", generator=g) if epi == 2 else None
    out = resid.clone() if epi == 2 else torch.empty(M, N, device="cuda")
    pg.linear_f32_device(A, W, bias, out, M, N, K, epi, out if epi == 2 else None)
    torch.cuda.synchronize()
    acc = A.double() @ W.double().t() + bias.double()
    if epi == 1:
        acc = 0.5 * acc * (1 + torch.erf(acc / 2 ** 0.5))
    if epi == 2:
        acc = resid.double() + acc
    scale = (A.double().abs() @ W.double().abs().t()) + bias.double().abs()
    err = ((out.double() - acc).abs() / (scale + 1e-30)).max().item()
    # the same GEMM in true fp32 (cuBLAS SGEMM, TF32 off): the summation-order noise floor
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    ref32 = (A @ W.t()).double() + bias.double()
    torch.backends.cuda.matmul.allow_tf32 = prev
    err32 = ((ref32 - (A.double() @ W.double().t() + bias.double())).abs() / (scale + 1e-30)).max().item()
    assert torch.isfinite(out).all()
    # measured: <= 2.6e-6 at K = 2048 (the tensor core's fp32 accumulation, ~6x the SGEMM
    # noise floor err32 ~ 4e-7; rounding the residues to nearest tf32 does not change it) --
    # 400x inside the fp32 policy's 1e-3 contract; a plain 1xTF32 GEMM sits near 1e-3
    assert err <= max(8 * err32, 5e-6), (err, err32)



# ---- fp32 logits straight from the head epilogue (EPI 5 = widened round16(acc)) ----
@pytest.mark.parametrize("M,N,ldo,bn,splits,lean", [
    (128, 30522, 30524, 0, 0, 0),     # C2/C3 head shape, 16-byte rows: TMA-store epilogue
    (256, 30522, 30522, 0, 0, 0),     # unaligned rows: per-thread stores
    (640, 50257, 50260, 256, 1, 2),   # CTA-pair kernel, M tail
    (200, 768, 768, 64, -3, 1),       # global-workspace split-K, lean pipeline
    (200, 768, 768, 128, 3, -1),      # (cluster split-K request: falls back to one split)
    (1, 96, 96, 0, 0, 0),
])
def test_tc_linear_f32_logits_match_f16(M, N, ldo, bn, splits, lean):
    """epi 5 writes exactly float(epi 3's fp16 value) into an fp32 buffer, on every kernel
    variant and store path, and leaves the pitch padding past the 16-byte chunk untouched."""
    K = 768
    g = torch.Generator(device="cuda").manual_seed(M + N)
    A = (torch.randn(M, K, device="cuda", generator=g) * 0.5).half()
    Wt = (torch.randn(N, K, device="cuda", generator=g) * 0.05).half()
    ld16 = (N + 7) // 8 * 8
    o16 = torch.empty(M, ld16, device="cuda", dtype=torch.float16)
    pg.linear_f16_device_ex(A, Wt, None, o16, M, N, K, ld16, 3, bn, splits, lean)
    o32 = torch.full((M, ldo), float("nan"), device="cuda", dtype=torch.float32)
    pg.linear_f16_device_ex(A, Wt, None, o32, M, N, K, ldo, 5, bn, splits, lean)
    torch.cuda.synchronize()
    assert torch.equal(o32[:, :N], o16[:, :N].float())
    # the TMA store writes whole 16-byte chunks: at most up to the next 4-float boundary
    assert torch.isnan(o32[:, (N + 3) // 4 * 4:]).all()
    with pytest.raises(ValueError):
        pg.linear_f16_device(A, Wt, None, o32, M, N, K, ldo, 4)  # row statistics: not an output epilogue


@pytest.mark.parametrize("B,S,causal", [(3, 384, 1), (5, 200, 0), (32, 512, 1), (1, 129, 1)])
def test_streaming_attention_dynamic_schedule(B, S, causal, monkeypatch):
    """The streaming kernel's dynamically claimed units (per-thread counter, re-armed by the
    last CTA of each launch) give the same ctx bit for bit as the static schedule, launch
    after launch, with shapes interleaved on the same counter."""
    H, hd = 12, 64
    g = torch.Generator(device="cuda").manual_seed(B * S + causal)
    qkv = (torch.randn(B * S, 3 * H * hd, device="cuda", generator=g) * 1.5).half()
    other = (torch.randn(2 * 256, 3 * H * hd, device="cuda", generator=g)).half()
    octx = torch.empty(2 * 256, H * hd, device="cuda", dtype=torch.float16)
    outs = []
    for _ in range(3):
        ctx = torch.full((B * S, H * hd), float("nan"), device="cuda", dtype=torch.float16)
        pg.attention_f16_device(qkv, ctx, B, S, H, hd, causal)
        pg.attention_f16_device(other, octx, 2, 256, H, hd, 1)  # another shape on the same counter
        outs.append(ctx)
    monkeypatch.setenv("PRLAB_ATTN_STATIC", "1")
    ref = torch.full((B * S, H * hd), float("nan"), device="cuda", dtype=torch.float16)
    pg.attention_f16_device(qkv, ref, B, S, H, hd, causal)
    torch.cuda.synchronize()
    assert torch.isfinite(ref.float()).all()
    for o in outs:
        assert torch.equal(o, ref)
