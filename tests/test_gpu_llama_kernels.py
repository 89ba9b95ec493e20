"""The LLaMA block's bandwidth kernels (llama_kernels.cu) and fused GEMM epilogues,
each pinned on its own against a plain PyTorch fp32 reference of the same op, at
every width the benchmarked workloads run (d = 512 / 1024 / 2048 select the
RMSNorm V4 = 4 / 8 / 16 instantiations; f = 2048 / 4096 / 5632; head_dim 64 and
128; T = 1024 / 4096) plus small and ragged cases.

Bars: fp32 outputs 1e-5 relative (max-norm) -- only the summation order differs;
bf16 outputs within one bf16 ulp of the fp32 reference (|err| <= 2^-7 |ref| +
1e-6, checked element-wise) unless the op rounds an intermediate, stated per test;
fused epilogues bit-identical to the separate kernels they replace.
"""
import math

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

EPS = 1e-5
BF16_REL = 2.0 ** -7  # one bf16 ulp (7 stored mantissa bits)


def _lib():
    from paper_2506_15461_b200._native import check, lib
    return check, lib()


def _close_bf16(got, want, rel=BF16_REL, atol=1e-6, ulps=1.0):
    got, want = got.float(), want.float()
    bad = (got - want).abs() > ulps * rel * want.abs() + atol
    assert not bad.any(), (int(bad.sum()), float((got - want).abs().max()))


def _rel_max(got, want):
    return float((got.double() - want.double()).abs().max() / want.double().abs().max().clamp_min(1e-30))


@pytest.mark.parametrize("d", [128, 256, 512, 1024, 2048])
@pytest.mark.parametrize("rows", [1, 37, 1000, 8192])
def test_rmsnorm_fwd_bwd(d, rows):
    check, L = _lib()
    g = torch.Generator(device="cuda").manual_seed(d * 7 + rows)
    x = torch.randn(rows, d, device="cuda", generator=g) * 3
    gain = 1 + 0.1 * torch.randn(d, device="cuda", generator=g)
    y = torch.empty(rows, d, device="cuda", dtype=torch.bfloat16)
    rstd = torch.empty(rows, device="cuda")
    xc = torch.empty_like(x)
    check(L.ckf_llama_rmsnorm_fwd(x.data_ptr(), gain.data_ptr(), rows, d, y.data_ptr(), rstd.data_ptr(),
                                  xc.data_ptr(), None))
    torch.cuda.synchronize()
    r_ref = torch.rsqrt((x.double() ** 2).mean(-1) + EPS)
    assert _rel_max(rstd, r_ref) < 1e-5
    assert torch.equal(xc, x)
    _close_bf16(y, (x.double() * r_ref[:, None] * gain.double()).float())
    # backward: dh += rstd (g dy - xhat mean(g dy xhat)); gg += sum_rows dy xhat
    dy = torch.randn(rows, d, device="cuda", generator=g)
    dh0 = torch.randn(rows, d, device="cuda", generator=g)
    dh = dh0.clone()
    dh_bf = torch.empty(rows, d, device="cuda", dtype=torch.bfloat16)
    gg0 = torch.randn(d, device="cuda", generator=g)
    gg = gg0.clone()
    check(L.ckf_llama_rmsnorm_bwd(dy.data_ptr(), x.data_ptr(), gain.data_ptr(), rstd.data_ptr(), rows, d,
                                  dh.data_ptr(), dh_bf.data_ptr(), gg.data_ptr(), None))
    torch.cuda.synchronize()
    xd, dyd, gd, rd = x.double(), dy.double(), gain.double(), rstd.double()[:, None]
    xhat = xd * rd
    gdy = gd * dyd
    dx = rd * (gdy - xhat * (gdy * xhat).mean(-1, keepdim=True))
    assert _rel_max(dh - dh0, dx) < 1e-5
    assert torch.equal(dh_bf, dh.bfloat16())
    assert _rel_max(gg - gg0, (dyd * xhat).sum(0)) < 1e-5


def _rope_ref(qkv, T, d, heads, inverse):
    hd = d // heads
    half = hd // 2
    ntok = qkv.shape[0]
    j = torch.arange(half, dtype=torch.float64, device=qkv.device)
    inv = 10000.0 ** (-2.0 * j / hd)
    pos = (torch.arange(ntok, device=qkv.device) % T).double()
    ang = pos[:, None] * inv[None, :]
    c, s = torch.cos(ang)[:, None, :], torch.sin(ang)[:, None, :]
    out = qkv.double().clone()
    for blk in (0, 1):  # q and k column blocks
        x = out[:, blk * d:(blk + 1) * d].reshape(ntok, heads, hd)
        x1, x2 = x[..., :half], x[..., half:]
        if inverse:
            y = torch.cat([x1 * c + x2 * s, x2 * c - x1 * s], -1)
        else:
            y = torch.cat([x1 * c - x2 * s, x2 * c + x1 * s], -1)
        out[:, blk * d:(blk + 1) * d] = y.reshape(ntok, d)
    return out


@pytest.mark.parametrize("T,d,heads", [(128, 256, 4), (1024, 512, 8), (1024, 1024, 16), (4096, 2048, 16)])
@pytest.mark.parametrize("inverse", [0, 1])
def test_rope(T, d, heads, inverse):
    check, L = _lib()
    g = torch.Generator(device="cuda").manual_seed(T + d)
    ntok = 2 * T
    qkv = torch.randn(ntok, 3 * d, device="cuda", generator=g).bfloat16()
    want = _rope_ref(qkv, T, d, heads, inverse)
    got = qkv.clone()
    check(L.ckf_llama_rope(got.data_ptr(), ntok, T, d, heads, inverse, None))
    torch.cuda.synchronize()
    # one bf16 rounding of an fp32 rotation (the fp32 cos/sin table adds ~1e-6 at t < 4096)
    _close_bf16(got[:, :2 * d], want[:, :2 * d].float(), atol=1e-3)
    assert torch.equal(got[:, 2 * d:], qkv[:, 2 * d:])  # v untouched


def _silu(x):
    return x * torch.sigmoid(x)


@pytest.mark.parametrize("f", [768, 2048, 4096, 5632])
def test_swiglu_fwd_bwd(f):
    check, L = _lib()
    g = torch.Generator(device="cuda").manual_seed(f)
    ntok = 1000
    gu = (torch.randn(ntok, 2 * f, device="cuda", generator=g) * 2).bfloat16()
    a = torch.empty(ntok, f, device="cuda", dtype=torch.bfloat16)
    check(L.ckf_llama_swiglu_fwd(gu.data_ptr(), ntok, f, a.data_ptr(), None))
    gg, uu = gu[:, :f].double(), gu[:, f:].double()
    da = torch.randn(ntok, f, device="cuda", generator=g).bfloat16()
    dgu = torch.empty(ntok, 2 * f, device="cuda", dtype=torch.bfloat16)
    check(L.ckf_llama_swiglu_bwd(gu.data_ptr(), da.data_ptr(), ntok, f, dgu.data_ptr(), None))
    torch.cuda.synchronize()
    _close_bf16(a, (_silu(gg) * uu).float(), atol=1e-5)
    sg = torch.sigmoid(gg)
    dd = da.double()
    _close_bf16(dgu[:, :f], (dd * uu * sg * (1 + gg * (1 - sg))).float(), atol=1e-5)
    _close_bf16(dgu[:, f:], (dd * _silu(gg)).float(), atol=1e-5)


@pytest.mark.parametrize("d,V", [(256, 4096), (512, 50304), (2048, 50304)])
def test_embedding_fwd_bwd(d, V):
    check, L = _lib()
    g = torch.Generator(device="cuda").manual_seed(d)
    ntok = 4096
    tok = torch.randint(0, V, (ntok,), device="cuda", generator=g, dtype=torch.int32)
    tok[::7] = 5  # repeated ids: the scatter must sum them in token order
    E = torch.randn(V, d, device="cuda", generator=g)
    h = torch.empty(ntok, d, device="cuda")
    check(L.ckf_llama_embed_fwd(tok.data_ptr(), ntok, E.data_ptr(), d, h.data_ptr(), None))
    torch.cuda.synchronize()
    assert torch.equal(h, E[tok.long()])
    dh = torch.randn(ntok, d, device="cuda", generator=g)
    gE = torch.randn(V, d, device="cuda", generator=g)
    gE0 = gE.clone()
    check(L.ckf_llama_embed_bwd(tok.data_ptr(), ntok, dh.data_ptr(), d, gE.data_ptr(), None))
    torch.cuda.synchronize()
    want = gE0.double().index_add(0, tok.long(), dh.double())
    assert _rel_max(gE, want) < 1e-5
    gE2 = gE0.clone()
    check(L.ckf_llama_embed_bwd(tok.data_ptr(), ntok, dh.data_ptr(), d, gE2.data_ptr(), None))
    torch.cuda.synchronize()
    assert torch.equal(gE, gE2)  # deterministic


def _gemm(M, N, K, A, a_mn, B, b_mn, C, ldc, epi, aux=None, ldaux=0):
    check, L = _lib()
    check(L.ckf_gemm_bf16_aux(M, N, K, A.data_ptr(), A.shape[1], int(a_mn), B.data_ptr(), B.shape[1], int(b_mn),
                              C.data_ptr(), ldc, epi, 1.0, 0, aux.data_ptr() if aux is not None else None, ldaux,
                              None))


@pytest.mark.parametrize("d,f", [(512, 2048), (1024, 4096), (2048, 5632)])
def test_fused_swiglu_epilogues_at_workload_widths(d, f):
    # forward gate/up GEMM with a = silu(g) u in its epilogue (epi 3) == GEMM + swiglu_fwd, bit for bit;
    # down-projection dgrad with dgu in its epilogue (epi 4) == GEMM (da) + swiglu_bwd, bit for bit;
    # both within bf16 rounding of the fp32 reference
    check, L = _lib()
    g = torch.Generator(device="cuda").manual_seed(f)
    M = 2048 + 64
    xn = (torch.randn(M, d, device="cuda", generator=g)).bfloat16()
    Wgu = (torch.randn(d, 2 * f, device="cuda", generator=g) / math.sqrt(d)).bfloat16()
    gu_f = torch.empty(M, 2 * f, device="cuda", dtype=torch.bfloat16)
    a_f = torch.empty(M, f, device="cuda", dtype=torch.bfloat16)
    _gemm(M, 2 * f, d, xn, False, Wgu, True, gu_f, 2 * f, 3, a_f, f)
    gu_s = torch.empty_like(gu_f)
    a_s = torch.empty_like(a_f)
    _gemm(M, 2 * f, d, xn, False, Wgu, True, gu_s, 2 * f, 0)
    check(L.ckf_llama_swiglu_fwd(gu_s.data_ptr(), M, f, a_s.data_ptr(), None))
    torch.cuda.synchronize()
    assert torch.equal(gu_f, gu_s) and torch.equal(a_f, a_s)
    ref = xn.float() @ Wgu.float()
    assert float((gu_f.float() - ref).norm() / ref.norm()) < 4e-3
    # backward: da = dh Wd^T (Wd [f x d] row-major = B K-major for N = f)
    dh = torch.randn(M, d, device="cuda", generator=g).bfloat16()
    Wd = (torch.randn(f, d, device="cuda", generator=g) / math.sqrt(f)).bfloat16()
    dgu_f = torch.empty(M, 2 * f, device="cuda", dtype=torch.bfloat16)
    _gemm(M, f, d, dh, False, Wd, False, dgu_f, 2 * f, 4, gu_f, 2 * f)
    da = torch.empty(M, f, device="cuda", dtype=torch.bfloat16)
    _gemm(M, f, d, dh, False, Wd, False, da, f, 0)
    dgu_s = torch.empty_like(dgu_f)
    check(L.ckf_llama_swiglu_bwd(gu_f.data_ptr(), da.data_ptr(), M, f, dgu_s.data_ptr(), None))
    torch.cuda.synchronize()
    assert torch.equal(dgu_f, dgu_s)
    da_ref = dh.float() @ Wd.float().t()
    assert float((da.float() - da_ref).norm() / da_ref.norm()) < 4e-3


@pytest.mark.parametrize("T,d,hd", [(1024, 512, 64), (1024, 1024, 64), (128, 256, 64), (4096, 2048, 128),
                                    (1024, 1024, 128), (256, 256, 128)])
def test_qkv_gemm_with_fused_rope(T, d, hd):
    # the QKV projection's epilogue applies RoPE to the fp32 accumulators before the bf16 store
    # (64-column heads: pairs inside one chunk; 128-column heads: pairs across a warp's two chunks):
    # within one bf16 rounding (plus the fp32 accumulation order) of the fp32 reference
    check, L = _lib()
    heads = d // hd
    g = torch.Generator(device="cuda").manual_seed(T + d)
    M = 2 * T
    A = torch.randn(M, d, device="cuda", generator=g).bfloat16()
    B = (torch.randn(d, 3 * d, device="cuda", generator=g) / math.sqrt(d)).bfloat16()
    C = torch.empty(M, 3 * d, device="cuda", dtype=torch.bfloat16)
    check(L.ckf_gemm_qkv_rope(M, d, A.data_ptr(), B.data_ptr(), C.data_ptr(), T, heads, None))
    torch.cuda.synchronize()
    want = _rope_ref((A.float() @ B.float()), T, d, heads, 0).float()
    err = float((C.float() - want).norm() / want.norm())
    assert err < 4e-3, err
    _close_bf16(C, want, ulps=2.0, atol=2e-2)
