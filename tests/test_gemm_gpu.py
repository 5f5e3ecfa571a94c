"""tcgen05 GEMM vs a plain PyTorch fp32 reference of the same contraction.

Tolerance: inputs are bf16 (exact in fp32), accumulation is fp32 in TMEM, so
the only error is the final bf16 rounding of the output (rel 2^-8) plus fp32
summation-order noise: |out - ref| <= 1e-2 * |ref| + 1e-2 * rms(ref).
fp32 outputs: |out - ref| <= 1e-4 * rms(ref) * sqrt(K/64) + 1e-5 * |ref|.
"""
import math

import pytest
import torch

pytestmark = pytest.mark.gpu


def _ops():
    from paper_2209_02478_b200 import ops
    return ops


def _check_bf16(out, ref):
    ref = ref.float()
    rms = ref.pow(2).mean().sqrt().item() + 1e-6
    err = (out.float() - ref).abs()
    bound = 1e-2 * ref.abs() + 1e-2 * rms
    assert torch.all(err <= bound), f"max err {err.max().item()} (rms {rms})"


def _check_f32(out, ref, K):
    rms = ref.pow(2).mean().sqrt().item() + 1e-6
    err = (out - ref).abs()
    bound = 1e-4 * rms * math.sqrt(max(K, 64) / 64) + 1e-5 * ref.abs()
    assert torch.all(err <= bound), f"max err {err.max().item()} (rms {rms})"


def _rand(*shape, dev="cuda"):
    return torch.randn(*shape, device=dev).to(torch.bfloat16)


@pytest.mark.parametrize("cg", [1, 2])
@pytest.mark.parametrize("ew", [8, 16])
@pytest.mark.parametrize("direct", [False, True])
@pytest.mark.parametrize("bn", [64, 128, 256])
@pytest.mark.parametrize("a_mn", [False, True])
@pytest.mark.parametrize("b_mn", [False, True])
@pytest.mark.parametrize("shape", [(256, 256, 128), (200, 72, 80), (1000, 770, 768), (128, 2304, 64)])
def test_gemm_majors(cuda_device, bn, a_mn, b_mn, shape, direct, ew, cg):
    if cg == 2 and (bn != 256 or shape[0] <= 128):
        pytest.skip("CTA pairs run 256-wide tiles with >= 2 row blocks")
    ops = _ops()
    torch.manual_seed(0)
    M, N, K = shape
    A = _rand(M, K)
    B = _rand(N, K)
    a_arg = A.t().contiguous() if a_mn else A
    b_arg = B.t().contiguous() if b_mn else B
    if (a_arg.stride(0) * 2) % 16 or (b_arg.stride(0) * 2) % 16:
        pytest.skip("TMA needs 16-byte row pitch")
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    ops.gemm(a_arg, b_arg, out, a_mn=a_mn, b_mn=b_mn, force_bn=bn, direct_store=direct,
             force_ew=ew, force_cg=cg)
    torch.cuda.synchronize()
    _check_bf16(out, A.float() @ B.float().t())


@pytest.mark.parametrize("cg", [1, 2])
@pytest.mark.parametrize("beta", [0.0, 0.5])
@pytest.mark.parametrize("bn", [128, 256])
def test_gemm_f32_beta(cuda_device, bn, beta, cg):
    ops = _ops()
    torch.manual_seed(1)
    M, N, K = 768, 3072, 4096
    # weight-gradient form: dW[N,K] = dY^T X with both operands MN-major
    dY = _rand(K, M)  # [T, N_out]
    X = _rand(K, N)   # [T, K_in]
    out = torch.randn(M, N, device="cuda")
    ref = out * beta + dY.float().t() @ X.float()
    ops.gemm(dY, X, out, a_mn=True, b_mn=True, epi=ops.EPI_F32, beta=beta, force_bn=bn,
             force_cg=cg)
    torch.cuda.synchronize()
    _check_f32(out, ref, K)


@pytest.mark.parametrize("cg", [1, 2])
@pytest.mark.parametrize("ew", [8, 16])
@pytest.mark.parametrize("M", [517, 1024])
def test_gemm_bias_gelu_and_dgelu(cuda_device, M, ew, cg):
    ops = _ops()
    torch.manual_seed(2)
    N, K = 3072, 768
    X = _rand(M, K)
    W = _rand(N, K) * 0.05
    bias = torch.randn(N, device="cuda")
    u = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    g = torch.empty_like(u)
    ops.gemm(X, W, u, epi=ops.EPI_BIAS_GELU, out2=g, bias=bias, force_ew=ew, force_cg=cg)
    torch.cuda.synchronize()
    u_ref = X.float() @ W.float().t() + bias
    _check_bf16(u, u_ref)
    g_ref = torch.nn.functional.gelu(u.float())
    assert torch.allclose(g.float(), g_ref, rtol=1e-2, atol=1e-2)

    # dGELU epilogue: out = (dY W) * gelu'(u)
    dY = _rand(M, K)
    du = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    W2 = _rand(K, N) * 0.05  # FFN2 weight [H, 4H]: dgrad B operand is MN-major view [K=H, N=4H]
    ops.gemm(dY, W2, du, b_mn=True, epi=ops.EPI_DGELU, aux=u, force_ew=ew, force_cg=cg)
    torch.cuda.synchronize()
    uf = u.float().requires_grad_(True)
    torch.nn.functional.gelu(uf).backward(torch.ones_like(uf))
    ref = (dY.float() @ W2.float()) * uf.grad
    _check_bf16(du, ref)


@pytest.mark.parametrize("S", [64, 128, 200, 512])
def test_gemm_attention_views(cuda_device, S):
    """Per-head batched views into a fused [B*S, 3H] QKV buffer (no copies)."""
    ops = _ops()
    torch.manual_seed(3)
    B, nh, d = 3, 12, 64
    H = nh * d
    qkv = _rand(B * S, 3 * H)
    q = qkv.view(B, S, 3, nh, d)[:, :, 0].permute(0, 2, 1, 3)  # [B, nh, S, d] strided
    k = qkv.view(B, S, 3, nh, d)[:, :, 1].permute(0, 2, 1, 3)
    v = qkv.view(B, S, 3, nh, d)[:, :, 2].permute(0, 2, 1, 3)
    ld = (S + 7) // 8 * 8
    scores_buf = torch.empty(B, nh, S, ld, device="cuda", dtype=torch.bfloat16)
    scores = scores_buf[..., :S]
    scale = 1.0 / math.sqrt(d)
    ops.gemm(q, k, scores, alpha=scale)
    torch.cuda.synchronize()
    ref = (q.float() @ k.float().transpose(-1, -2)) * scale
    _check_bf16(scores, ref)

    # ctx = P V with V MN-major (d contiguous), written head-interleaved into [B*S, H]
    P = torch.softmax(ref, -1).to(torch.bfloat16)
    Pbuf = torch.zeros(B, nh, S, ld, device="cuda", dtype=torch.bfloat16)
    Pbuf[..., :S] = P
    ctx = torch.empty(B * S, H, device="cuda", dtype=torch.bfloat16)
    ctx_v = ctx.view(B, S, nh, d).permute(0, 2, 1, 3)
    ops.gemm(Pbuf[..., :S], v, ctx_v, b_mn=True)
    torch.cuda.synchronize()
    _check_bf16(ctx_v, P.float() @ v.float())

    # dV = P^T dO (both MN-major), dK = dS^T Q
    dO = _rand(B, nh, S, d)
    dV = torch.empty(B, nh, S, d, device="cuda", dtype=torch.bfloat16)
    ops.gemm(Pbuf[..., :S], dO, dV, a_mn=True, b_mn=True)
    torch.cuda.synchronize()
    _check_bf16(dV, P.float().transpose(-1, -2) @ dO.float())


def test_gemm_residual_aux_add(cuda_device):
    """bf16 epilogue with a residual: out = A B^T + aux (gradient sums)."""
    ops = _ops()
    torch.manual_seed(4)
    M, N, K = 700, 768, 3072
    A = _rand(M, K)
    B = _rand(N, K) * 0.05
    aux = _rand(M, N)
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    ops.gemm(A, B, out, aux=aux)
    torch.cuda.synchronize()
    _check_bf16(out, A.float() @ B.float().t() + aux.float())


@pytest.mark.parametrize("split", [0, 2, 4, 7])
@pytest.mark.parametrize("shape", [(768, 768, 18432), (2304, 768, 4096), (104, 200, 1000)])
def test_gemm_wgrad_split_k(cuda_device, split, shape):
    """Deterministic split-K (fp32 partials + fixed-order reduce) for weight grads."""
    ops = _ops()
    torch.manual_seed(5)
    M, N, K = shape
    dY = _rand(K, M)
    X = _rand(K, N)
    ws = torch.empty(8 * M * N, device="cuda")
    out = torch.empty(M, N, device="cuda")
    ops.gemm(dY, X, out, a_mn=True, b_mn=True, epi=ops.EPI_F32, split_k=split, workspace=ws)
    out2 = torch.empty_like(out)
    ops.gemm(dY, X, out2, a_mn=True, b_mn=True, epi=ops.EPI_F32, split_k=split, workspace=ws)
    torch.cuda.synchronize()
    _check_f32(out, dY.float().t() @ X.float(), K)
    assert torch.equal(out, out2)  # run-to-run bitwise


@pytest.mark.parametrize("roomy", [True, False])
@pytest.mark.parametrize("cg", [0, 1, 2])
@pytest.mark.parametrize("split", [0, 1, 2, 5])
@pytest.mark.parametrize("shape", [(3072, 768, 18432), (2304, 768, 4096), (104, 200, 1000),
                                   (768, 3072, 2560)])
def test_gemm_wgrad_rowsum(cuda_device, cg, split, shape, roomy):
    """Weight gradient + bias gradient in one GEMM: the row-sum warps' sums of
    the staged dY tiles equal dY's column sums (fp32 over the same bf16
    values), dW is bitwise the GEMM without them, and both are run-to-run
    bitwise. roomy: the workspace holds a row-sum partial per column tile
    (every tile sums a share of the k-blocks); tight: only per split (the
    first column tile sums them all)."""
    ops = _ops()
    torch.manual_seed(11)
    M, N, K = shape
    if cg == 2 and M <= 128:
        pytest.skip("CTA pairs need M > 128")
    dY = _rand(K, M)
    X = _rand(K, N)
    ws = torch.empty(8 * M * (N + (N + 63) // 64) if roomy else 8 * M * N + 8 * M, device="cuda")
    kw = dict(a_mn=True, b_mn=True, epi=ops.EPI_F32, split_k=split, workspace=ws, force_cg=cg,
              force_bn=256 if cg == 2 else 0)
    ref_w = torch.empty(M, N, device="cuda")
    ops.gemm(dY, X, ref_w, **kw)
    outs = []
    for _ in range(2):
        w = torch.empty(M, N, device="cuda")
        db = torch.full((M,), float("nan"), device="cuda")
        ops.gemm(dY, X, w, rowsum=db, **kw)
        outs.append((w, db))
    torch.cuda.synchronize()
    ref_b = dY.double().sum(0)
    for w, db in outs:
        assert torch.equal(w, ref_w)
        err = (db.double() - ref_b).abs()
        bound = 2e-6 * dY.double().abs().sum(0) + 1e-6
        assert torch.all(err <= bound), f"max err {err.max().item()}"
    assert torch.equal(outs[0][1], outs[1][1])


def test_gemm_rowsum_rejects_unsupported(cuda_device):
    ops = _ops()
    A, B = _rand(256, 128), _rand(192, 128)
    db = torch.empty(256, device="cuda")
    with pytest.raises(Exception):  # K-major A has no row-sum path
        ops.gemm(A, B, torch.empty(256, 192, device="cuda"), epi=ops.EPI_F32, rowsum=db)
    with pytest.raises(Exception):  # bf16 epilogues neither
        ops.gemm(A.t().contiguous(), B, torch.empty(256, 192, device="cuda", dtype=torch.bfloat16),
                 a_mn=True, rowsum=db)
