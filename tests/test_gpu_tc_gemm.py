"""The tensor-core GEMM behind the tiny-MLP head (csrc/tc_gemm.cu: tcgen05.mma
kind::tf32, 3-term hi/lo split, TMEM accumulators) against fp64 numpy, for the
operand orders and tile widths the head uses. Bar: every entry within
4e-6 * sum_l |a_il b_jl| (fp32-class: ~2^-21 per product plus fp32
accumulation), i.e. far inside the 1e-4 north-star tolerance."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("image", [0, 1])
@pytest.mark.parametrize("m,n,k,ak,bk", [
    (128, 16, 32, True, True), (300, 3, 25, True, True), (1000, 256, 256, True, True),
    (777, 64, 200, True, False), (256, 256, 4096, False, False), (129, 33, 65, False, True),
    (65536, 256, 256, True, True), (300, 300, 70, True, True)])
def test_tc_gemm_matches_fp64(m, n, k, ak, bk, image):
    import torch

    from paper_2405_16788_b200._lib import check, lib

    rng = np.random.default_rng(m + n + k)
    a = rng.standard_normal((m, k)).astype(np.float32)
    b = rng.standard_normal((n, k)).astype(np.float32)
    a_dev = torch.from_numpy(a if ak else np.ascontiguousarray(a.T)).cuda()
    b_dev = torch.from_numpy(b if bk else np.ascontiguousarray(b.T)).cuda()
    d = torch.full((m, n), np.nan, dtype=torch.float32, device="cuda")
    torch.cuda.synchronize()
    check(lib().dpl_gemm_f32(0, None, m, n, k, a_dev.data_ptr(), k if ak else m, int(ak),
                             b_dev.data_ptr(), k if bk else n, int(bk), d.data_ptr(), n, image))
    got = d.cpu().numpy().astype(np.float64)
    ref = a.astype(np.float64) @ b.astype(np.float64).T
    mag = np.abs(a).astype(np.float64) @ np.abs(b).astype(np.float64).T
    err = np.abs(got - ref)
    bad = ~(err <= 4e-6 * mag + 1e-30)
    assert not bad.any(), (int(bad.sum()), float((err / mag).max()))
