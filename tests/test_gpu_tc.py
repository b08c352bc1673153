"""Tensor-core building blocks (tcgen05.mma kind::f16 via csrc/tc.cuh) against exact
references: the fp16 products are exact in fp32, so a single MMA must match the float64
dot product of the fp16 inputs to fp32 accumulation error; subnormal fp16 inputs must
not be flushed; the 3-pass hi/lo split must reach fp32-class accuracy."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def pack(M: np.ndarray) -> np.ndarray:
    """Canonical no-swizzle K-major packing (csrc/tc.cuh canon_idx) of an R x K fp16 matrix."""
    R, K = M.shape
    out = np.empty(R * K, dtype=np.float16)
    r = np.arange(R)[:, None]
    k = np.arange(K)[None, :]
    idx = (((r >> 3) * (K >> 3) + (k >> 3)) << 6) + ((r & 7) << 3) + (k & 7)
    out[idx.reshape(-1)] = M.reshape(-1)
    return out


@pytest.fixture(scope="module")
def ctx():
    from paper_2202_13638_b200 import bagel

    return bagel.Context(0)


def _run(ctx, A16, B16, mode=0):
    N, K = B16.shape
    a16 = pack(A16) if mode == 0 else np.ascontiguousarray(A16)
    a = torch.from_numpy(a16.view(np.int16).reshape(-1)).cuda()
    b = torch.from_numpy(pack(B16).view(np.int16)).cuda()
    return ctx.tc_selftest(a, b, N, K, mode).cpu().numpy().astype(np.float64)


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("N,K", [(256, 64), (16, 16), (128, 128), (32, 512), (272 - 16, 32)])
def test_single_mma_matches_exact_products(ctx, N, K, mode):
    """mode 0: A and B from shared memory; mode 1: A from TMEM (TS form)."""
    if mode == 1 and N + K // 2 > 512:
        pytest.skip("TMEM columns")
    rng = np.random.default_rng(N * 1000 + K)
    A = rng.uniform(-1, 1, (128, K)).astype(np.float16)
    B = rng.uniform(-1, 1, (N, K)).astype(np.float16)
    D = _run(ctx, A, B, mode)
    ref = A.astype(np.float64) @ B.astype(np.float64).T
    scale = np.abs(A.astype(np.float64)) @ np.abs(B.astype(np.float64)).T
    assert np.all(np.abs(D - ref) <= 4 * K * 2.0 ** -24 * scale + 1e-30)


def test_subnormal_fp16_inputs_are_not_flushed(ctx):
    A = np.zeros((128, 16), dtype=np.float16)
    A[:, 0] = np.float16(2.0 ** -20)  # subnormal in fp16 (min normal 2^-14)
    A[:, 1] = np.float16(3 * 2.0 ** -24)
    B = np.zeros((16, 16), dtype=np.float16)
    B[:, 0] = 1.0
    B[:, 1] = 2.0
    D = _run(ctx, A, B)
    assert np.allclose(D, 2.0 ** -20 + 6 * 2.0 ** -24, rtol=1e-6, atol=0)


def test_three_pass_split_reaches_fp32_accuracy(ctx):
    """a = a_hi + a_lo, b = b_hi + b_lo (fp16 each); a.b ~ a_hi b_hi + a_hi b_lo + a_lo b_hi."""
    rng = np.random.default_rng(7)
    K, N = 256, 256
    a = np.exp2(-rng.uniform(0, 12, (128, K))).astype(np.float32)      # ktilde-like, (0, 1]
    b = (rng.normal(size=(N, K)) * np.exp2(-rng.uniform(0, 4, (N, 1)))).astype(np.float32)
    a_hi = a.astype(np.float16)
    a_lo = (a - a_hi.astype(np.float32)).astype(np.float16)
    b_hi = b.astype(np.float16)
    b_lo = (b - b_hi.astype(np.float32)).astype(np.float16)
    D = _run(ctx, a_hi, b_hi) + _run(ctx, a_hi, b_lo) + _run(ctx, a_lo, b_hi)
    ref = a.astype(np.float64) @ b.astype(np.float64).T
    scale = np.abs(a.astype(np.float64)) @ np.abs(b.astype(np.float64)).T
    err = np.abs(D - ref) / scale
    print("3-pass max error / sum|a b|:", err.max(), " (2^-24 =", 2.0 ** -24, ")")
    assert err.max() < 64 * 2.0 ** -24


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("N,K", [(256, 64), (128, 32), (64, 128), (128, 256)])
def test_cta_pair_mma_matches_exact_products(ctx, N, K, mode):
    """tcgen05.mma.cta_group::2 (M = 256 over a 2-CTA cluster): A rows 0-127 / 128-255 live in the
    leader's / peer's shared memory (mode 0) or TMEM (mode 1, the TS form), B columns 0..N/2-1 /
    N/2..N-1 in the leader's / peer's shared memory; D rows land in each CTA's TMEM."""
    if mode == 1 and N + K // 2 > 512:
        pytest.skip("TMEM columns")
    rng = np.random.default_rng(N + K)
    A = rng.uniform(-1, 1, (256, K)).astype(np.float16)
    B = rng.uniform(-1, 1, (N, K)).astype(np.float16)
    a = torch.from_numpy(np.concatenate([pack(A[:128]), pack(A[128:]), A.reshape(-1)]).view(np.int16)).cuda()
    b = torch.from_numpy(np.concatenate([pack(B[: N // 2]), pack(B[N // 2:])]).view(np.int16)).cuda()
    D = ctx.tc_selftest2(a, b, N, K, mode).cpu().numpy().astype(np.float64)
    ref = A.astype(np.float64) @ B.astype(np.float64).T
    scale = np.abs(A.astype(np.float64)) @ np.abs(B.astype(np.float64)).T
    assert np.all(np.abs(D - ref) <= 4 * K * 2.0 ** -24 * scale + 1e-30), np.abs(D - ref).max()
