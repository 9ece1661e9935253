"""tcgen05 (5th-generation tensor core) encodings: qs_probe_umma runs
D = A @ B (128 x 128 x 128, bf16 operands, fp32 accumulate in TMEM) with the
operands staged K-major or MN-major in the blocked no-swizzle layout the fused
critic kernel uses, against a host matmul of the same bf16-rounded inputs."""

import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("mode", [0, 1, 2, 3])
def test_umma_descriptors_match_matmul(mode):
    from paper_2509_10247_b200 import _lib as L

    g = torch.Generator().manual_seed(mode)
    A = torch.randn(128, 128, generator=g).cuda()
    B = torch.randn(128, 128, generator=g).cuda()
    D = torch.zeros(128, 128, device="cuda")
    L.check(L.lib().qs_probe_umma(mode, L.ptr(A), L.ptr(B), L.ptr(D), L.stream_handle()), "qs_probe_umma")
    ref = A.bfloat16().float() @ B.bfloat16().float()
    err = (D - ref).abs().max().item() / ref.abs().max().item()
    assert err < 1e-5, (mode, err)
