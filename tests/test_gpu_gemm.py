"""Decode-GEMM tiers against a plain f32/f64 reference of the same op
(the numerics check for a floating-point kernel): tier 1 (CUDA cores) and
tier 2 (tcgen05 + TMA + TMEM), every epilogue, split-K and odd N tails."""
import numpy as np
import pytest

from paper_2504_10724_b200 import eeb

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    c = eeb.Context(0)
    yield c
    c.close()


def ref_gemm(w, x, mode):
    y = (x.astype(np.float64) @ w.astype(np.float64).T)
    if mode == 2:
        y = np.maximum(y, 0)
    if mode == 3:
        g, u = y[:, 0::2], y[:, 1::2]
        y = g / (1 + np.exp(-g)) * u
    return y


@pytest.mark.parametrize("tier", [1, 2])
@pytest.mark.parametrize("n,k,b", [(128, 256, 16), (2048, 2048, 64), (6144, 2048, 64), (2048, 8192, 32),
                                   (50272, 2048, 64), (1000, 512, 48), (4096, 1024, 256), (2048, 2048, 4),
                                   (1000, 512, 3), (2048, 2048, 200), (6144, 2048, 130),
                                   # long K above 128 rows: one 256-column tile per weight tile (deep)
                                   (2048, 8192, 256), (1000, 8192, 176)])
@pytest.mark.parametrize("mode", [0, 2, 3])
def test_gemm_tiers(ctx, tier, n, k, b, mode):
    if tier == 1 and b > 64:
        pytest.skip("tier 1 serves <= 64 rows")
    if mode == 3 and n % 2:
        pytest.skip()
    rng = np.random.default_rng(n + k + b + mode)
    w = eeb.bf16_round(rng.standard_normal((n, k)).astype(np.float32) * 0.02)
    x = eeb.bf16_round(rng.standard_normal((b, k)).astype(np.float32))
    y = ctx.debug_gemm(tier, w, x, mode)
    r = ref_gemm(w, x, mode)
    if mode >= 2:   # bf16-rounded outputs
        np.testing.assert_allclose(y, r, rtol=1e-2, atol=1e-2 * np.abs(r).max())
    else:
        np.testing.assert_allclose(y, r, rtol=1e-4, atol=1e-4 * np.abs(r).max())
