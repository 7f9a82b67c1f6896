"""Kernel-isolated numerics of the tcgen05 verify GEMM against a plain fp64 PyTorch CPU reference
of the same op (out = X W^T, and the fused SwiGLU dual GEMM)."""
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

SHAPES = [  # (M tokens, N weight rows, K) — several tiles, ragged tails, split-K/stream-K cuts
    (1, 128, 256), (4, 512, 256), (16, 6144, 4096), (20, 688, 256), (16, 4096, 14336), (64, 1280, 1024),
    (128, 256, 688), (256, 1024, 512), (48, 128256 // 8, 4096),
]


def _ref(X, W, M):
    return X[:M].double().cpu() @ W.double().cpu().T


@pytest.mark.parametrize("M,N,K", SHAPES)
def test_gemm_matches_fp64_reference(M, N, K):
    from paper_2409_03856_b200 import sirius as S
    g = torch.Generator(device="cpu").manual_seed(M * 7 + N + K)
    rows = max(16, (M + 15) // 16 * 16)
    X = (torch.randn(rows, K, generator=g) * 0.5).to(torch.bfloat16).cuda()
    W = (torch.randn(N, K, generator=g) / K ** 0.5).to(torch.bfloat16).cuda()
    out = torch.full((M, N), float("nan"), dtype=torch.float32, device="cuda")
    S.debug_gemm(X, W, out, M)
    ref = _ref(X, W, M)
    err = (out.double().cpu() - ref).abs()
    # fp32 accumulation of K bf16 products: |err| <= K * 2^-24 * sum|x w| (generous bound used: 1e-5 * sqrt(K) scale)
    bound = 2e-6 * K ** 0.5 * 4 + 1e-5 * ref.abs()
    assert torch.isfinite(out).all()
    assert (err <= bound).all(), float(err.max())


def _split3(x32):
    """fp32 -> three bf16 terms t0 + t1 + t2 == x32 exactly (the library's split3, D15a)."""
    t0 = x32.to(torch.bfloat16)
    r1 = x32 - t0.float()
    t1 = r1.to(torch.bfloat16)
    t2 = (r1 - t1.float()).to(torch.bfloat16)
    return torch.stack([t0, t1, t2])


def test_split3_is_exact():
    x = torch.randn(100000) * 10.0 ** torch.randint(-8, 8, (100000,)).float()
    t = _split3(x)
    assert torch.equal(t[0].double() + t[1].double() + t[2].double(), x.double())


@pytest.mark.parametrize("M,N,K", [(16, 14336 // 8, 4096), (5, 688, 256), (64, 512, 1024)])
def test_dual_swiglu_gemm_fp32_activations(M, N, K):
    """Dual gate/up GEMM with fp32 activations fed as three bf16 terms; m = SiLU(g) u comes back as
    three bf16 terms: agrees with fp64 on the fp32 inputs to fp32 accumulation error."""
    from paper_2409_03856_b200 import sirius as S
    g = torch.Generator(device="cpu").manual_seed(1 + M + N)
    X32 = torch.randn(256, K, generator=g)
    W1 = (torch.randn(N, K, generator=g) / K ** 0.5).to(torch.bfloat16).cuda()
    W2 = (torch.randn(N, K, generator=g) / K ** 0.5).to(torch.bfloat16).cuda()
    m3 = torch.zeros((3, M, N), dtype=torch.bfloat16, device="cuda")
    S.debug_gemm(_split3(X32).cuda(), W1, m3, M, W2=W2)
    x = X32[:M].double()
    gte = x @ W1.double().cpu().T
    up = x @ W2.double().cpu().T
    ref = gte / (1 + torch.exp(-gte)) * up
    got = m3.double().cpu().sum(0)
    err = (got - ref).abs()
    assert (err <= 2e-6 * ref.abs() + 4e-6 * K ** 0.5 * 0.05).all(), float(err.max())


def test_gemm_split3_is_fp32_grade():
    """out = (t0 + t1 + t2) W^T matches fp64 on the fp32 activations to fp32 accumulation error (not
    just on bf16(X): that would be ~1e-2; the earlier two-term split gave ~1e-4)."""
    from paper_2409_03856_b200 import sirius as S
    g = torch.Generator(device="cpu").manual_seed(11)
    M, N, K = 16, 1024, 4096
    X32 = torch.randn(16, K, generator=g)
    W = (torch.randn(N, K, generator=g) / K ** 0.5).to(torch.bfloat16).cuda()
    out = torch.zeros((M, N), dtype=torch.float32, device="cuda")
    S.debug_gemm(_split3(X32).cuda(), W, out, M)
    ref = X32.double() @ W.double().cpu().T
    err = (out.double().cpu() - ref).abs()
    assert float(err.max()) < 2e-5, float(err.max())


def test_gemm_deterministic():
    from paper_2409_03856_b200 import sirius as S
    X = torch.randn(16, 4096).to(torch.bfloat16).cuda()
    W = (torch.randn(4096, 4096) / 64).to(torch.bfloat16).cuda()
    a = torch.empty((16, 4096), device="cuda")
    b = torch.empty((16, 4096), device="cuda")
    S.debug_gemm(X, W, a, 16)
    S.debug_gemm(X, W, b, 16)
    assert torch.equal(a, b)
