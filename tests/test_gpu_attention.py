"""Causal attention kernels against a plain PyTorch fp32 reference of the same op
(softmax(q k^T / sqrt(hd)) v with a causal mask, RoPE already applied upstream).
Bars: outputs 2e-2 relative Frobenius error (bf16 operands and P), lse 1e-3 abs,
gradients 3e-2 relative per q / k / v block.  Both forward implementations
(mma.sync flash, tcgen05/TMEM) are checked, and they must agree with each other."""
import math

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _ref(qkv, B, T, H, hd):
    x = qkv.float().view(B, T, 3, H, hd)
    q, k, v = x[:, :, 0].transpose(1, 2), x[:, :, 1].transpose(1, 2), x[:, :, 2].transpose(1, 2)
    s = q @ k.transpose(-1, -2) / math.sqrt(hd)
    mask = torch.triu(torch.ones(T, T, dtype=torch.bool, device=qkv.device), 1)
    s = s.masked_fill(mask, float("-inf"))
    lse = torch.logsumexp(s, -1)
    o = torch.softmax(s, -1) @ v
    return o.transpose(1, 2).reshape(B * T, H * hd), lse.reshape(B * H * T)


def _fwd(qkv, B, T, H, hd, impl):
    from paper_2506_15461_b200._native import check, lib
    o = torch.empty(B * T, H * hd, dtype=torch.bfloat16, device="cuda")
    lse = torch.empty(B * H * T, device="cuda")
    check(lib().ckf_attention_fwd(qkv.data_ptr(), B, T, H, hd, o.data_ptr(), lse.data_ptr(), impl, None))
    torch.cuda.synchronize()
    return o, lse


@pytest.mark.parametrize("impl", [1, 2])
@pytest.mark.parametrize("shape", [(2, 128, 2, 64), (2, 256, 3, 64), (1, 1024, 2, 64), (2, 128, 2, 128),
                                   (2, 1024, 2, 128)])
def test_forward_vs_torch(impl, shape):
    B, T, H, hd = shape
    if impl == 2 and (hd not in (64, 128) or T % 128):
        pytest.skip("tcgen05 kernel: hd 64 or 128, T % 128")
    import paper_2506_15461_b200  # noqa: F401
    torch.manual_seed(0)
    qkv = (torch.randn(B * T, 3 * H * hd, device="cuda") * 0.8).bfloat16()
    o, lse = _fwd(qkv, B, T, H, hd, impl)
    ro, rl = _ref(qkv, B, T, H, hd)
    assert ((o.float() - ro).norm() / ro.norm()).item() < 2e-2
    assert (lse - rl).abs().max().item() < 1e-3 * max(1.0, rl.abs().max().item())


@pytest.mark.parametrize("hd", [64, 128])
def test_forward_rising_scores_rescale_paths(hd):
    """Scores that grow along the key axis (k_t = (1 + t/2) * a shared direction, q along it
    too): every later 64-key tile beats the running max, which exercises the redo of a tile
    against its own max and the lazy O / l rescale (the fast path keeps P <= 2^16)."""
    import paper_2506_15461_b200  # noqa: F401
    torch.manual_seed(3)
    B, T, H = 1, 1024, 2
    dirn = torch.randn(hd, device="cuda")
    dirn = dirn / dirn.norm()
    x = torch.randn(B * T, 3, H, hd, device="cuda") * 0.3
    ramp = 1.0 + torch.arange(T, device="cuda", dtype=torch.float32) / 2.0  # ~23 log2 units per 64 keys
    x[:, 0] += 4.0 * dirn  # q along the shared direction
    x[:, 1] += ramp[:, None, None] * dirn  # k grows along it
    qkv = x.reshape(B * T, 3 * H * hd).bfloat16()
    o, lse = _fwd(qkv, B, T, H, hd, 2)
    ro, rl = _ref(qkv, B, T, H, hd)
    assert torch.isfinite(o.float()).all()
    assert ((o.float() - ro).norm() / ro.norm()).item() < 2e-2
    assert ((lse - rl).abs() / rl.abs().clamp(min=1.0)).max().item() < 1e-3


def test_tcgen05_matches_mma_sync():
    import paper_2506_15461_b200  # noqa: F401
    torch.manual_seed(1)
    B, T, H, hd = 4, 1024, 4, 64
    qkv = torch.randn(B * T, 3 * H * hd, device="cuda").bfloat16()
    o1, l1 = _fwd(qkv, B, T, H, hd, 1)
    o2, l2 = _fwd(qkv, B, T, H, hd, 2)
    assert ((o1.float() - o2.float()).norm() / o1.float().norm()).item() < 1e-2
    assert (l1 - l2).abs().max().item() < 1e-3
    # deterministic
    o3, l3 = _fwd(qkv, B, T, H, hd, 2)
    assert torch.equal(o2, o3) and torch.equal(l2, l3)


@pytest.mark.parametrize("impl", [1, 2])
@pytest.mark.parametrize("shape", [(2, 128, 2, 64), (1, 512, 2, 64), (2, 1024, 2, 64), (1, 512, 2, 128),
                                   (2, 1024, 3, 128)])
def test_backward_vs_torch(shape, impl):
    from paper_2506_15461_b200._native import check, lib
    B, T, H, hd = shape
    if impl == 2 and hd not in (64, 128):
        pytest.skip("tcgen05 kernel: hd 64 or 128")
    torch.manual_seed(2)
    qkv = (torch.randn(B * T, 3 * H * hd, device="cuda") * 0.8).bfloat16()
    o, lse = _fwd(qkv, B, T, H, hd, 0)
    dout = torch.randn(B * T, H * hd, device="cuda").bfloat16()
    dqkv = torch.zeros(B * T, 3 * H * hd, dtype=torch.bfloat16, device="cuda")
    Dsum = torch.empty(B * H * T, device="cuda")
    check(lib().ckf_attention_bwd(qkv.data_ptr(), o.data_ptr(), lse.data_ptr(), dout.data_ptr(), B, T, H, hd,
                                  dqkv.data_ptr(), Dsum.data_ptr(), impl, None))
    torch.cuda.synchronize()
    x = qkv.float().requires_grad_(True)
    ro, _ = _ref(x, B, T, H, hd)
    ro.backward(dout.float())
    g = x.grad
    for blk in range(3):
        a = dqkv.float()[:, blk * H * hd:(blk + 1) * H * hd]
        b = g[:, blk * H * hd:(blk + 1) * H * hd]
        assert ((a - b).norm() / b.norm()).item() < 3e-2, blk


@pytest.mark.parametrize("shape", [(2, 256, 2, 64), (1, 1024, 3, 64), (1, 512, 2, 128), (1, 1024, 2, 128)])
def test_backward_with_fused_rope_inverse(shape):
    """impl | CKF_ATTN_ROPE_BWD (16): the dK / dQ epilogues apply the RoPE backward in fp32 before the
    single bf16 rounding.  Checked against the fp32-torch attention gradient rotated by the
    fp64 inverse RoPE (3e-2 per block, as the plain backward) and against the unfused
    backward + ckf_llama_rope pass (two roundings: 1e-2); dv must be bit-identical to the plain
    backward (no rotation on v)."""
    from paper_2506_15461_b200._native import check, lib
    from test_gpu_llama_kernels import _rope_ref
    B, T, H, hd = shape
    torch.manual_seed(5)
    qkv = (torch.randn(B * T, 3 * H * hd, device="cuda") * 0.8).bfloat16()
    o, lse = _fwd(qkv, B, T, H, hd, 0)
    dout = torch.randn(B * T, H * hd, device="cuda").bfloat16()
    Dsum = torch.empty(B * H * T, device="cuda")
    fused = torch.zeros(B * T, 3 * H * hd, dtype=torch.bfloat16, device="cuda")
    plain = torch.zeros_like(fused)
    check(lib().ckf_attention_bwd(qkv.data_ptr(), o.data_ptr(), lse.data_ptr(), dout.data_ptr(), B, T, H, hd,
                                  fused.data_ptr(), Dsum.data_ptr(), 2 | 16, None))
    check(lib().ckf_attention_bwd(qkv.data_ptr(), o.data_ptr(), lse.data_ptr(), dout.data_ptr(), B, T, H, hd,
                                  plain.data_ptr(), Dsum.data_ptr(), 2, None))
    torch.cuda.synchronize()
    d = H * hd
    assert torch.equal(fused[:, 2 * d:], plain[:, 2 * d:])
    two = plain.clone()
    check(lib().ckf_llama_rope(two.data_ptr(), B * T, T, d, H, 1, None))
    x = qkv.float().requires_grad_(True)
    ro, _ = _ref(x, B, T, H, hd)
    ro.backward(dout.float())
    want = _rope_ref(x.grad.detach(), T, d, H, 1).float()
    for blk in range(2):
        a = fused.float()[:, blk * d:(blk + 1) * d]
        b = want[:, blk * d:(blk + 1) * d]
        c = two.float()[:, blk * d:(blk + 1) * d]
        assert ((a - b).norm() / b.norm()).item() < 3e-2, blk
        assert ((a - c).norm() / c.norm()).item() < 1e-2, blk


@pytest.mark.parametrize("M,d,hd,T", [(2048, 1024, 64, 1024), (1024, 512, 64, 256), (4096, 2048, 128, 4096),
                                       (512, 256, 128, 256)])
def test_o_dgrad_gemm_with_fused_dsum(M, d, hd, T):
    """The O-projection dgrad's epilogue forms the attention backward's D = rowsum(bf16(dO) . O) per
    head: dO within one bf16 rounding of fp32 torch, D against torch's sum over the same bf16
    operands (fp32 summation-order differences only: 1e-4 relative to the row's |dO| |O|)."""
    from paper_2506_15461_b200._native import check, lib
    g = torch.Generator(device="cuda").manual_seed(M + d)
    A = torch.randn(M, d, generator=g, device="cuda").bfloat16()
    W = (torch.randn(d, d, generator=g, device="cuda") / d ** 0.5).bfloat16()  # Wo stored [K][N]
    O = torch.randn(M, d, generator=g, device="cuda").bfloat16()
    C = torch.empty(M, d, dtype=torch.bfloat16, device="cuda")
    H = d // hd
    D = torch.full((M // T * H * T,), float("nan"), device="cuda")
    check(lib().ckf_gemm_o_dgrad_dsum(M, d, A.data_ptr(), W.data_ptr(), C.data_ptr(), O.data_ptr(), D.data_ptr(),
                                      T, H, None))
    torch.cuda.synchronize()
    want = A.float() @ W.float().t()
    assert float((C.float() - want).norm() / want.norm()) < 4e-3
    prod = (C.float() * O.float()).view(M // T, T, H, hd)
    Dw = prod.sum(-1).permute(0, 2, 1).reshape(-1)
    scale = (C.float().abs() * O.float().abs()).view(M // T, T, H, hd).sum(-1).permute(0, 2, 1).reshape(-1)
    assert torch.isfinite(D).all()
    assert float(((D - Dw).abs() / scale.clamp_min(1e-6)).max()) < 1e-4


_CHUNK_SCRIPT = r"""
import sys, torch
sys.path.insert(0, sys.argv[1])
import paper_2506_15461_b200  # noqa: F401
from paper_2506_15461_b200._native import check, lib
B, T, H, hd = (int(v) for v in sys.argv[2:6])
torch.manual_seed(5)
qkv = (torch.randn(B * T, 3 * H * hd, device="cuda") * 0.8).bfloat16()
o = torch.empty(B * T, H * hd, dtype=torch.bfloat16, device="cuda")
lse = torch.empty(B * H * T, device="cuda")
check(lib().ckf_attention_fwd(qkv.data_ptr(), B, T, H, hd, o.data_ptr(), lse.data_ptr(), 2, None))
dout = torch.randn(B * T, H * hd, device="cuda").bfloat16()
dqkv = torch.zeros(B * T, 3 * H * hd, dtype=torch.bfloat16, device="cuda")
D = torch.empty(B * H * T, device="cuda")
check(lib().ckf_attention_bwd(qkv.data_ptr(), o.data_ptr(), lse.data_ptr(), dout.data_ptr(), B, T, H, hd,
                              dqkv.data_ptr(), D.data_ptr(), 0, None))
torch.cuda.synchronize()
torch.save(dqkv.cpu(), sys.argv[6])
"""


@pytest.mark.parametrize("shape", [(3, 512, 2, 64), (3, 512, 2, 128)])
def test_backward_one_pass_per_sequence_is_bit_identical(shape, tmp_path):
    """The stored-dS backward runs in passes of as many sequences as the causal dS^T scratch
    budget holds (CKF_ATTN_DS_BYTES, read once per process).  A budget below one sequence forces a
    pass per sequence; each sequence's arithmetic is the same either way, so dq / dk / dv must be
    bit-identical to the single-pass run."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for budget in (None, "1"):
        env = dict(os.environ)
        env.pop("CKF_ATTN_DS_BYTES", None)
        if budget:
            env["CKF_ATTN_DS_BYTES"] = budget
        path = str(tmp_path / f"dqkv_{budget}.pt")
        subprocess.run([sys.executable, "-c", _CHUNK_SCRIPT, root, *map(str, shape), path], env=env, check=True,
                       timeout=600)
        outs.append(torch.load(path))
    assert torch.equal(outs[0], outs[1])
    assert outs[0].float().abs().sum().item() > 0


_FWD_SCRIPT = r"""
import sys, torch
sys.path.insert(0, sys.argv[1])
import paper_2506_15461_b200  # noqa: F401
from paper_2506_15461_b200._native import check, lib
outs = []
for (B, T, H, hd) in [(1, 128, 1, 64), (3, 1024, 5, 64), (2, 512, 3, 128), (8, 1024, 8, 64), (8, 1024, 12, 128),
                      (1, 128, 1, 64), (3, 1024, 5, 64)]:
    torch.manual_seed(B * 1000 + T + H + hd)
    qkv = (torch.randn(B * T, 3 * H * hd, device="cuda") * 0.8).bfloat16()
    o = torch.empty(B * T, H * hd, dtype=torch.bfloat16, device="cuda")
    lse = torch.empty(B * H * T, device="cuda")
    check(lib().ckf_attention_fwd(qkv.data_ptr(), B, T, H, hd, o.data_ptr(), lse.data_ptr(), 2, None))
    torch.cuda.synchronize()
    outs.append((o.cpu(), lse.cpu()))
torch.save(outs, sys.argv[2])
"""


def test_forward_persistent_ctas_bit_identical_to_one_cta_per_unit(tmp_path):
    """The persistent forward (CTAs drawing units from a counter that the last CTA resets) against
    one CTA per unit (CKF_ATTN_FWD_PERSIST=0, read once per process): a unit's arithmetic is the
    same either way, so outputs and lse are bit-identical -- over a launch sequence with fewer
    units than CTAs, more units than CTAs, both head dims, and repeated shapes (a counter left
    non-zero by one launch would skip units of the next)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = []
    for persist in ("1", "0"):
        env = dict(os.environ)
        env["CKF_ATTN_FWD_PERSIST"] = persist
        path = str(tmp_path / f"fwd_{persist}.pt")
        subprocess.run([sys.executable, "-c", _FWD_SCRIPT, root, path], env=env, check=True, timeout=600)
        res.append(torch.load(path))
    for (o1, l1), (o0, l0) in zip(*res):
        assert torch.equal(o1, o0) and torch.equal(l1, l0)
    assert torch.equal(res[0][0][0], res[0][5][0]) and torch.equal(res[0][1][0], res[0][6][0])


@pytest.mark.parametrize("shape", [(8, 1024, 8, 64), (8, 1024, 12, 128)])
def test_forward_many_units_per_persistent_cta(shape):
    """More (sequence x head, query tile) units than persistent CTAs (512 on 296 at hd 64, 384
    two-tile units on 148 at hd 128): each CTA runs several units back to back -- S / P buffer
    and K / V stage phases carried across units, Q reloaded under the previous unit's softmax, O
    handed back between units, and at hd 128 the second tile's extra K / V tiles released by the
    first group too.  Checked against the fp32 reference."""
    B, T, H, hd = shape
    import paper_2506_15461_b200  # noqa: F401
    torch.manual_seed(7)
    qkv = (torch.randn(B * T, 3 * H * hd, device="cuda") * 0.8).bfloat16()
    o, lse = _fwd(qkv, B, T, H, hd, 2)
    ro, rl = _ref(qkv, B, T, H, hd)
    assert ((o.float() - ro).norm() / ro.norm()).item() < 2e-2
    assert (lse - rl).abs().max().item() < 1e-3 * max(1.0, rl.abs().max().item())
