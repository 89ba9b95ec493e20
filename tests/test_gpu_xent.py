"""LLaMA head loss kernel (llama_kernels.cu xent_bf16, via ckf_xent_bf16) against a plain PyTorch
fp32 reference of the same op: row loss = logsumexp(logits) - logits[label], gradient =
grad_scale * (softmax - onehot) written over the bf16 logits.  Covers the persistent
row-pipelined kernel (V = 50304, the LLaMA vocabulary) and the register kernel (small V)."""
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("rows,V", [(300, 50304), (64, 512), (37, 4096)])
def test_xent_bf16_matches_torch_fp32(rows, V):
    from paper_2506_15461_b200._native import check, lib

    g = torch.Generator(device="cuda").manual_seed(rows + V)
    logits = (torch.randn(rows, V, device="cuda", generator=g) * 3.0).bfloat16()
    labels = torch.randint(0, V, (rows,), device="cuda", generator=g, dtype=torch.int32)
    ref_x = logits.float()
    lse = torch.logsumexp(ref_x, dim=1)
    ref_loss = lse - ref_x.gather(1, labels.long()[:, None])[:, 0]
    scale = 1.0 / rows
    ref_grad = (torch.softmax(ref_x, dim=1) - torch.nn.functional.one_hot(labels.long(), V).float()) * scale

    row_loss = torch.zeros(rows, device="cuda", dtype=torch.float64)
    work = logits.clone()
    check(lib().ckf_xent_bf16(work.data_ptr(), labels.data_ptr(), rows, V, scale, 1, row_loss.data_ptr(), None))
    torch.cuda.synchronize()
    # loss: fp32 accumulation with approximate exp2 (MUFU ~2 ulp, FMA polynomial < 3e-6 rel)
    assert torch.allclose(row_loss.float(), ref_loss, rtol=2e-5, atol=2e-5), (row_loss.float() - ref_loss).abs().max()
    # gradient: one bf16 rounding of the fp32 value (2^-8 relative) plus the exp error
    err = (work.float() - ref_grad).abs()
    tol = ref_grad.abs() * (2.0 ** -8) + 1e-6 * scale
    assert (err <= tol).all(), (err - tol).max()

    # loss only (grad = 0): logits untouched
    row2 = torch.zeros_like(row_loss)
    keep = logits.clone()
    check(lib().ckf_xent_bf16(keep.data_ptr(), labels.data_ptr(), rows, V, scale, 0, row2.data_ptr(), None))
    torch.cuda.synchronize()
    assert torch.equal(keep, logits)
    assert torch.equal(row2, row_loss)
