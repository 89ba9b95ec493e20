"""tcgen05 bf16 GEMM (gemm_tc.cu) against a plain PyTorch fp32 reference of the same op.

Covers every operand layout the stage forward / dgrad / wgrad use (A and B
each K-major or MN-major), all three epilogues, both N tiles, and ragged
M / N / K tails (TMA zero-fill + epilogue bounds).  Tolerances: fp32 epilogues
1e-3 relative Frobenius error (only the fp32 summation order differs); bf16
store 8e-3 (one bf16 rounding of the result).
"""
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _ref(A, B, M, N, K, a_mn, b_mn):
    a = (A.float().t() if a_mn else A.float())[:M, :K]
    b = (B.float() if b_mn else B.float().t())[:K, :N]
    return a @ b


def _run(M, N, K, a_mn, b_mn, epi, bn=0, alpha=1.0, seed=0):
    import paper_2506_15461_b200 as P
    from paper_2506_15461_b200._native import check, lib
    g = torch.Generator(device="cuda").manual_seed(seed)
    def ld(x):  # padded row pitch, a multiple of 8 elements (16-byte TMA pitch)
        return (x + 8 + 7) // 8 * 8
    A = (torch.randn((K, ld(M)) if a_mn else (M, ld(K)), generator=g, device="cuda") * 0.5).bfloat16()
    B = (torch.randn((K, ld(N)) if b_mn else (N, ld(K)), generator=g, device="cuda") * 0.5).bfloat16()
    ldc = ld(N)
    if epi == 0:
        C = torch.zeros((M, ldc), dtype=torch.bfloat16, device="cuda")
    else:
        C = torch.randn((M, ldc), generator=g, device="cuda") if epi == 2 else torch.zeros((M, ldc), device="cuda")
    C0 = C.clone()
    check(lib().ckf_gemm_bf16(M, N, K, A.data_ptr(), A.shape[1], int(a_mn), B.data_ptr(), B.shape[1], int(b_mn),
                              C.data_ptr(), ldc, epi, alpha, bn, None))
    torch.cuda.synchronize()
    want = alpha * _ref(A, B, M, N, K, a_mn, b_mn)
    if epi == 2:
        want = want + C0[:, :N].float()
    got = C[:, :N].float()
    err = (got - want).norm() / want.norm()
    # untouched padding columns
    assert torch.equal(C[:, N:], C0[:, N:])
    return err.item()


@pytest.mark.parametrize("a_mn", [False, True])
@pytest.mark.parametrize("b_mn", [False, True])
@pytest.mark.parametrize("epi", [0, 1, 2])
def test_layouts_and_epilogues(a_mn, b_mn, epi):
    err = _run(256, 512, 512, a_mn, b_mn, epi)
    assert err < (8e-3 if epi == 0 else 1e-3), err


@pytest.mark.parametrize("shape", [(128, 128, 64), (300, 200, 136), (1000, 384, 1000), (64, 96, 40)])
@pytest.mark.parametrize("bn", [128, 256])
def test_ragged_tails(shape, bn):
    M, N, K = shape
    for a_mn, b_mn in ((False, True), (False, False), (True, True)):
        err = _run(M, N, K, a_mn, b_mn, 1, bn=bn)
        assert err < 1e-3, (shape, a_mn, b_mn, err)


def test_stage_shapes_and_alpha():
    # LLaMA-124M stage GEMMs at M_tok = 8192: QKV fwd, down-proj dgrad, QKV wgrad
    assert _run(8192, 1536, 512, False, True, 0) < 8e-3
    assert _run(8192, 2048, 512, False, False, 1, alpha=0.5) < 1e-3
    assert _run(512, 1536, 8192, True, True, 2) < 1e-3


@pytest.mark.parametrize("shape", [(300, 200, 2000), (512, 512, 8192), (2048, 512, 8192), (512, 4096, 16384),
                                   (512, 1536, 65536), (384, 640, 4096)])
def test_split_k_accumulate(shape):
    # few output tiles + long K -> split-K (CTA pairs when M >= 256) with an ordered, deterministic
    # workspace reduction
    M, N, K = shape
    assert _run(M, N, K, True, True, 2) < 1e-3


def test_split_k_deterministic():
    import paper_2506_15461_b200  # noqa: F401
    from paper_2506_15461_b200._native import check, lib
    A = torch.randn(8192, 512, device="cuda").bfloat16()
    B = torch.randn(8192, 1536, device="cuda").bfloat16()
    outs = []
    for _ in range(3):
        C = torch.ones(512, 1536, device="cuda")
        check(lib().ckf_gemm_bf16(512, 1536, 8192, A.data_ptr(), 512, 1, B.data_ptr(), 1536, 1, C.data_ptr(), 1536, 2,
                                  1.0, 0, None))
        outs.append(C)
    torch.cuda.synchronize()
    assert torch.equal(outs[0], outs[1]) and torch.equal(outs[1], outs[2])


def test_deterministic():
    import paper_2506_15461_b200  # noqa: F401
    from paper_2506_15461_b200._native import check, lib
    A = torch.randn(2048, 1024, device="cuda").bfloat16()
    B = torch.randn(1024, 768, device="cuda").bfloat16()
    outs = []
    for _ in range(3):
        C = torch.zeros(2048, 768, device="cuda")
        check(lib().ckf_gemm_bf16(2048, 768, 1024, A.data_ptr(), 1024, 0, B.data_ptr(), 768, 1, C.data_ptr(), 768, 1,
                                  1.0, 0, None))
        outs.append(C)
    torch.cuda.synchronize()
    assert torch.equal(outs[0], outs[1]) and torch.equal(outs[1], outs[2])
