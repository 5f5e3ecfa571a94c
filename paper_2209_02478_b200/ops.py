"""Thin torch-facing wrappers over the C-ABI device operators (tests/bench).

torch is only plumbing here (device buffers, streams); all arithmetic runs in
the sm_100a kernels of libmimose_cuda.so.
"""
from __future__ import annotations

import ctypes as C

import torch

from ._lib import GemmArgs, check, cuda_lib

EPI_BF16, EPI_BIAS_GELU, EPI_DGELU, EPI_F32 = 0, 1, 2, 3


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _view(t: torch.Tensor, nb1: int, nb2: int):
    """Describe a bf16 tensor as (ptr, rows, cols, ld, bs1, bs2).

    Accepts 2-D [rows, cols] (nb1 = nb2 = 1), 3-D [nb1, rows, cols] and
    4-D [nb2, nb1, rows, cols] strided views with a contiguous last dim.
    """
    assert t.dtype == torch.bfloat16 and t.stride(-1) == 1
    if t.dim() == 2:
        return t.data_ptr(), t.shape[0], t.shape[1], t.stride(0), 0, 0
    if t.dim() == 3:
        assert t.shape[0] == nb1 and nb2 == 1
        return t.data_ptr(), t.shape[1], t.shape[2], t.stride(1), t.stride(0), 0
    assert t.dim() == 4 and t.shape[0] == nb2 and t.shape[1] == nb1
    return t.data_ptr(), t.shape[2], t.shape[3], t.stride(2), t.stride(1), t.stride(0)


def gemm(a, b, out, *, a_mn=False, b_mn=False, epi=EPI_BF16, out2=None, aux=None, bias=None,
         alpha=1.0, beta=0.0, force_bn=0, force_ew=0, force_cg=0, direct_store=False, split_k=1,
         workspace=None, rowsum=None, stream=None):
    """out[z] = alpha * op(a)[z] @ op(b)[z]^T with the kernel's epilogue.

    a: [.., M, K] (a_mn False) or [.., K, M] (a_mn True); b: [.., N, K] or [.., K, N].
    out: [.., M, N] (bf16, or fp32 for EPI_F32).
    rowsum: fp32 [M] (EPI_F32, a_mn, unbatched): also the sums of op(a)'s rows
    over K (the bias gradient of a weight gradient).
    """
    nb2 = out.shape[0] if out.dim() == 4 else 1
    nb1 = out.shape[-3] if out.dim() >= 3 else 1
    M, N = out.shape[-2], out.shape[-1]
    pa = _view(a, nb1, nb2)
    pb = _view(b, nb1, nb2)
    K = pa[1] if a_mn else pa[2]
    assert (pb[1] if b_mn else pb[2]) == K
    args = GemmArgs()
    args.M, args.N, args.K, args.nb1, args.nb2 = M, N, K, nb1, nb2
    args.a, args.a_rows, args.a_cols, args.lda, args.a_bs1, args.a_bs2 = pa
    args.a_mn = int(a_mn)
    args.b, args.b_rows, args.b_cols, args.ldb, args.b_bs1, args.b_bs2 = pb
    args.b_mn = int(b_mn)
    args.epi = epi
    args.out = out.data_ptr()
    args.out2 = out2.data_ptr() if out2 is not None else None
    args.aux = aux.data_ptr() if aux is not None else None
    args.bias = bias.data_ptr() if bias is not None else None
    args.ldo = out.stride(-2)
    args.obs1 = out.stride(-3) if out.dim() >= 3 else 0
    args.obs2 = out.stride(0) if out.dim() == 4 else 0
    args.alpha, args.beta = alpha, beta
    args.force_bn = force_bn
    args.force_ew = force_ew
    args.force_cg = force_cg
    args.direct_store = int(direct_store)
    args.split_k = split_k
    if workspace is not None:
        args.workspace = workspace.data_ptr()
        args.workspace_bytes = workspace.numel() * workspace.element_size()
    if rowsum is not None:
        assert rowsum.dtype == torch.float32 and rowsum.numel() == M
        args.rowsum = rowsum.data_ptr()
    lib = cuda_lib()
    check(lib.mimose_gemm(C.byref(args), _stream(stream)))
    return out


def _attn_args(qkv, B, S, nh, causal, dropout_p, seed, stream_id, scale):
    from ._lib import AttnArgs
    assert qkv.dtype == torch.bfloat16 and qkv.is_contiguous() and qkv.shape == (B * S, 3 * 64 * nh)
    a = AttnArgs()
    a.B, a.S, a.nh, a.causal = B, S, nh, int(causal)
    a.scale, a.dropout_p = scale, dropout_p
    a.seed, a.stream_id = seed, stream_id
    a.qkv = qkv.data_ptr()
    return a


def flash_attn_fwd(qkv, B, S, nh, *, causal=False, dropout_p=0.0, seed=0, stream_id=0,
                   scale=0.125, stream=None):
    """Flash attention forward over packed qkv [B*S, 3H] (head dim 64).
    Returns (ctx [B*S, H] bf16, lse [B*nh, S] fp32 log2-sum-exp of the scaled scores,
    keep mask [B*nh*S, ceil(S/32)] int32 bits or None without dropout)."""
    H = 64 * nh
    ctx = torch.empty(B * S, H, device=qkv.device, dtype=torch.bfloat16)
    lse = torch.empty(B * nh, S, device=qkv.device, dtype=torch.float32)
    mask = (torch.empty(B * nh * S, (S + 31) // 32, device=qkv.device, dtype=torch.int32)
            if dropout_p > 0 else None)
    a = _attn_args(qkv, B, S, nh, causal, dropout_p, seed, stream_id, scale)
    a.ctx, a.lse = ctx.data_ptr(), lse.data_ptr()
    a.keep_mask = mask.data_ptr() if mask is not None else None
    check(cuda_lib().mimose_flash_attn_fwd(C.byref(a), _stream(stream)))
    return ctx, lse, mask


def flash_attn_bwd(qkv, ctx, lse, mask, dctx, B, S, nh, *, causal=False, dropout_p=0.0, seed=0,
                   stream_id=0, scale=0.125, stream=None):
    """Flash attention backward: dqkv [B*S, 3H] from dctx and the forward's ctx / lse."""
    dqkv = torch.empty_like(qkv)
    ws = torch.empty(B * nh * S, device=qkv.device, dtype=torch.float32)
    a = _attn_args(qkv, B, S, nh, causal, dropout_p, seed, stream_id, scale)
    a.ctx, a.lse, a.dctx, a.dqkv = ctx.data_ptr(), lse.data_ptr(), dctx.data_ptr(), dqkv.data_ptr()
    a.keep_mask = mask.data_ptr() if mask is not None else None
    a.workspace, a.workspace_bytes = ws.data_ptr(), ws.numel() * 4
    check(cuda_lib().mimose_flash_attn_bwd(C.byref(a), _stream(stream)))
    return dqkv
