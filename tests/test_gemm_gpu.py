"""Linear-layer kernels vs a plain torch fp32 reference (K5): the tcgen05 GEMM in both operand
orders (normal / swap-AB, split-K), the small-batch dgemv path and the TMA-ring tgemv path,
with every fused epilogue."""
import pytest
import torch

from paper_2603_10342_b200.device import debug_gemm

pytestmark = pytest.mark.gpu

EPI_BF16, EPI_RESID, EPI_SILU, EPI_F32 = 0, 1, 2, 3


def _ref(x, w, bias, resid, epi):
    acc = x.float() @ w.float().t()
    if epi == EPI_BF16:
        if bias is not None:
            acc = acc + bias.float()
        return acc
    if epi == EPI_RESID:
        return acc + resid.float()
    if epi == EPI_SILU:
        g, u = acc[:, 0::2], acc[:, 1::2]
        return torch.nn.functional.silu(g) * u
    return acc


@pytest.mark.parametrize("T,N,K,path,splits", [
    (300, 896, 896, 0, 0), (1024, 1152, 896, 0, 0), (2048, 4096, 512, 0, 0),
    (8, 1152, 896, 1, 0), (80, 896, 4864, 1, 0), (33, 4096, 1024, 1, 1), (200, 512, 256, 1, 3),
    (130, 256, 704, 0, 0), (1, 4096, 256, 1, 0),
    # cluster split-K at >= 32 tokens: bulk-push reduction (ragged N, odd token counts)
    (64, 3072, 1024, 1, 5), (45, 1000, 640, 1, 6), (32, 896, 896, 1, 7),
    # path 2: small-batch dgemv (legacy warp MMA fed from HBM), T <= 32, ragged N
    (1, 4096, 256, 2, 0), (8, 1152, 896, 2, 0), (13, 896, 4864, 2, 0), (16, 9728, 896, 2, 0),
    (24, 512, 256, 2, 0), (32, 1000, 640, 2, 0), (5, 136, 3072, 2, 0),
    # path 3: tgemv (TMA smem ring + warp MMA), T <= 32: chosen K splits, forced splits with the
    # last-arriver reduction, ragged N, an odd k-block count (half-OOB last k-unit)
    (1, 4096, 256, 3, 0), (8, 1152, 896, 3, 0), (13, 896, 4864, 3, 0), (16, 9728, 896, 3, 0),
    (24, 512, 256, 3, 0), (32, 1000, 640, 3, 0), (5, 136, 3072, 3, 0), (17, 3072, 3072, 3, 4),
    (31, 1000, 704, 3, 3), (9, 256, 8192, 3, 8),
])
@pytest.mark.parametrize("epi", [EPI_BF16, EPI_RESID, EPI_SILU, EPI_F32])
def test_gemm(T, N, K, path, splits, epi):
    torch.manual_seed(T * 7 + N + K + epi)
    dev = "cuda"
    x = (torch.randn(T, K, device=dev) * 0.5).bfloat16()
    w = (torch.randn(N, K, device=dev) * 0.05).bfloat16()
    bias = (torch.randn(N, device=dev) * 0.1).bfloat16() if epi == EPI_BF16 else None
    resid = (torch.randn(T, N, device=dev)).bfloat16() if epi == EPI_RESID else None
    if epi == EPI_F32:
        out = torch.zeros(T, N, device=dev, dtype=torch.float32)
    elif epi == EPI_SILU:
        out = torch.zeros(T, N // 2, device=dev, dtype=torch.bfloat16)
    elif epi == EPI_RESID:
        out = resid.clone()  # in-place residual add, as the forward uses it
    else:
        out = torch.zeros(T, N, device=dev, dtype=torch.bfloat16)
    ref = _ref(x, w, bias, resid, epi)
    torch.cuda.synchronize()
    debug_gemm(x.data_ptr(), w.data_ptr(), out.data_ptr(), T, N, K, epi,
               bias=bias.data_ptr() if bias is not None else None,
               resid=out.data_ptr() if resid is not None else None,
               force_path=path, splits=splits)
    got = out.float()
    err = (got - ref).abs().max().item()
    scale = ref.abs().max().item() + 1e-6
    # bf16 output rounding (2^-8 relative) plus fp32 summation-order noise
    tol = 1e-4 * scale if epi == EPI_F32 else 8e-3 * scale
    assert err <= tol, f"max abs err {err} vs tol {tol} (scale {scale})"
