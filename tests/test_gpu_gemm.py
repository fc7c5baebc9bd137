"""GEMM parity on the B200 (-m gpu): the tcgen05 kernel in every operand
majorness, bf16 and 3xTF32, ragged shapes spanning several tiles, split-K,
bias/ReLU/beta epilogues — against the oracle's float64 matmul."""
import numpy as np
import pytest

from gpu_common import be_init, rel
from oracle import ops
from oracle.autograd import Var

pytestmark = pytest.mark.gpu


def _ref(a, b, ta, tb, bias=None, act=0, beta=0.0, d0=None):
    A = a.T if ta else a
    B = b.T if tb else b
    y = ops.matmul(Var(A.astype(np.float64)), Var(B.astype(np.float64))).value
    if bias is not None:
        y = y + bias
    if act:
        y = np.maximum(y, 0)
    if beta:
        y = y + d0
    return y


@pytest.mark.parametrize("dtype,tol", [("bf16", 1e-2), ("f32", 1e-5)])
@pytest.mark.parametrize("ta,tb", [(0, 0), (0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("M,N,K", [(128, 128, 64), (300, 200, 136), (1024, 512, 512), (64, 40, 3000)])
def test_gemm_majorness(dtype, tol, ta, tb, M, N, K):
    be = be_init()
    rng = np.random.default_rng(M + N + K + ta * 2 + tb)
    a = rng.standard_normal((K, M) if ta else (M, K)).astype(np.float32)
    b = rng.standard_normal((N, K) if tb else (K, N)).astype(np.float32)
    if dtype == "bf16":  # compare against the bf16-rounded operands (the kernel's inputs)
        from paper_1912_01703_b200.api import f32_to_bf16_bits, bf16_bits_to_f32
        a = bf16_bits_to_f32(f32_to_bf16_bits(a))
        b = bf16_bits_to_f32(f32_to_bf16_bits(b))
    A = be.tensor(a, dtype=dtype)
    B = be.tensor(b, dtype=dtype)
    D = be.empty((M, N), "f32")
    be.gemm(A, B, D, trans_a=bool(ta), trans_b=bool(tb))
    ref = _ref(a, b, ta, tb)
    e = rel(D.numpy(), ref)
    assert e < (1e-5 if dtype == "bf16" else tol), e


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_gemm_epilogue_bias_relu_beta(dtype):
    be = be_init()
    rng = np.random.default_rng(7)
    M, N, K = 257, 384, 192
    a = rng.standard_normal((M, K)).astype(np.float32)
    b = rng.standard_normal((K, N)).astype(np.float32)
    bias = rng.standard_normal(N).astype(np.float32)
    d0 = rng.standard_normal((M, N)).astype(np.float32)
    if dtype == "bf16":
        from paper_1912_01703_b200.api import f32_to_bf16_bits, bf16_bits_to_f32
        a = bf16_bits_to_f32(f32_to_bf16_bits(a))
        b = bf16_bits_to_f32(f32_to_bf16_bits(b))
    A, B = be.tensor(a, dtype=dtype), be.tensor(b, dtype=dtype)
    D = be.tensor(d0)
    be.gemm(A, B, D, bias=be.tensor(bias), act=1, beta=1.0)
    ref = _ref(a, b, 0, 0, bias, 1, 1.0, d0)
    assert rel(D.numpy(), ref) < (1e-5 if dtype == "bf16" else 2e-6)
    # bf16 output, RN-even rounding of the fp32 accumulator
    Db = be.empty((M, N), "bf16")
    be.gemm(A, B, Db)
    assert rel(Db.numpy(), _ref(a, b, 0, 0)) < 8e-3


def test_gemm_splitk_deterministic():
    """Split-K (tiny M·N, huge K) reduces partials in a fixed order."""
    be = be_init()
    rng = np.random.default_rng(3)
    M, N, K = 64, 147, 60000
    a = rng.standard_normal((K, M)).astype(np.float32)
    b = rng.standard_normal((K, N)).astype(np.float32)
    A, B = be.tensor(a, dtype="bf16"), be.tensor(b, dtype="bf16")
    D1, D2 = be.empty((M, N), "f32"), be.empty((M, N), "f32")
    for _ in range(24):  # let the per-shape autotuner (which cycles its candidate kernels) settle
        be.gemm(A, B, D1, trans_a=True)
        be.synchronize()
    be.gemm(A, B, D1, trans_a=True)
    be.gemm(A, B, D2, trans_a=True)
    x1, x2 = D1.numpy(), D2.numpy()
    assert np.array_equal(x1, x2)
    from paper_1912_01703_b200.api import f32_to_bf16_bits, bf16_bits_to_f32
    ab = bf16_bits_to_f32(f32_to_bf16_bits(a)).astype(np.float64)
    bb = bf16_bits_to_f32(f32_to_bf16_bits(b)).astype(np.float64)
    assert rel(x1, ab.T @ bb) < 1e-5


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("M,N,K,ta,tb", [(64, 10, 128, 0, 0), (300, 10, 84, 0, 1), (37, 1000, 10, 1, 0),
                                         (129, 3, 5, 0, 0)])
def test_gemm_misaligned_operands_padded(M, N, K, ta, tb, dtype):
    """Operands whose rows are not 16-byte multiples (the N = 10 heads of C1
    and the smoke MLP) are padded into temporaries so the product stays on
    the tcgen05 kernel; every kernel the op launches is one of ours (no SIMT
    fallback), the result matches float64."""
    be = be_init()
    rng = np.random.default_rng(M + N + K)
    a = rng.standard_normal((K, M) if ta else (M, K)).astype(np.float32)
    b = rng.standard_normal((N, K) if tb else (K, N)).astype(np.float32)
    if dtype == "bf16":
        from paper_1912_01703_b200.api import f32_to_bf16_bits, bf16_bits_to_f32
        a = bf16_bits_to_f32(f32_to_bf16_bits(a))
        b = bf16_bits_to_f32(f32_to_bf16_bits(b))
    D = be.empty((M, N), "f32")
    be.gemm(be.tensor(a, dtype=dtype), be.tensor(b, dtype=dtype), D, trans_a=bool(ta), trans_b=bool(tb))
    assert rel(D.numpy(), _ref(a, b, ta, tb)) < 1e-5


_EPI4_SCRIPT = r'''
import sys, numpy as np
sys.path[:0] = [sys.argv[1], sys.argv[1] + "/tests"]
import paper_1912_01703_b200 as be
from paper_1912_01703_b200.api import f32_to_bf16_bits, bf16_bits_to_f32
be.init(0)
worst = 0.0
for (M, N, K, out, beta, act) in [(148 * 128 + 77, 256, 64, "bf16", 0.0, 0), (148 * 128 * 2, 128, 128, "f32", 0.0, 1),
                                  (148 * 128 + 5, 64, 200, "bf16", 1.0, 0), (148 * 128, 1024, 256, "bf16", 0.0, 1)]:
    rng = np.random.default_rng(M + N)
    a = bf16_bits_to_f32(f32_to_bf16_bits(rng.standard_normal((M, K)).astype(np.float32)))
    b = bf16_bits_to_f32(f32_to_bf16_bits(rng.standard_normal((N, K)).astype(np.float32)))
    bias = rng.standard_normal(N).astype(np.float32)
    d0 = bf16_bits_to_f32(f32_to_bf16_bits(rng.standard_normal((M, N)).astype(np.float32)))
    D = be.tensor(d0, dtype=out if out == "bf16" else None)
    be.gemm(be.tensor(a, dtype="bf16"), be.tensor(b, dtype="bf16"), D, trans_b=True, bias=be.tensor(bias),
            act=act, beta=beta)
    ref = a.astype(np.float64) @ b.T.astype(np.float64) + bias
    if act:
        ref = np.maximum(ref, 0)
    ref = ref + beta * d0
    e = float(np.abs(D.numpy() - ref).max() / np.abs(ref).max())
    worst = max(worst, e)
print(worst)
'''


def test_gemm_four_slot_epilogue(tmp_path):
    """The 4-slot (3 TMA stores in flight per warp) epilogue variant of the
    1-CTA kernel, forced with BE_GEMM_EPI4=1 on short-K store-heavy shapes
    (ragged M, bf16 / fp32 out, bias, ReLU, beta = 1 reduce-add store), vs
    float64 at the storage rounding of the output (2^-8 relative for bf16)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    f = tmp_path / "epi4.py"
    f.write_text(_EPI4_SCRIPT)
    env = dict(os.environ, BE_GEMM_EPI4="1")
    out = subprocess.run([sys.executable, str(f), root], env=env, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    assert float(out.stdout.strip().splitlines()[-1]) < 8e-3


@pytest.mark.parametrize("M,N,K,act,beta,out", [(50000, 16, 96, 0, 0.0, "bf16"), (40000, 24, 144, 1, 0.0, "bf16"),
                                                (30011, 64, 32, 0, 1.0, "bf16"), (20000, 40, 70, 1, 0.0, "f32"),
                                                (60000, 144, 24, 0, 0.0, "bf16"), (9000, 200, 64, 1, 1.0, "f32")])
def test_gemm_narrow_outputs_tile_split_epilogue(M, N, K, act, beta, out):
    """Narrow outputs (BN = 64: the tile-split epilogue, each warp pair taking
    alternate tiles) and ragged N on wider tiles (interleaved 64-column
    pieces), many tiles per CTA, bias / ReLU / beta-accumulate, bf16 and fp32
    outputs — vs float64 at the output's storage rounding."""
    be = be_init()
    rng = np.random.default_rng(M + N + K)
    from paper_1912_01703_b200.api import f32_to_bf16_bits, bf16_bits_to_f32
    q = lambda a: bf16_bits_to_f32(f32_to_bf16_bits(a.astype(np.float32)))  # noqa: E731
    a, b = q(rng.standard_normal((M, K))), q(rng.standard_normal((N, K)))
    bias = rng.standard_normal(N).astype(np.float32)
    d0 = q(rng.standard_normal((M, N)))
    D = be.tensor(d0, dtype=out if out == "bf16" else None)
    be.gemm(be.tensor(a, dtype="bf16"), be.tensor(b, dtype="bf16"), D, trans_b=True, bias=be.tensor(bias), act=act,
            beta=beta)
    ref = a.astype(np.float64) @ b.T.astype(np.float64) + bias
    if act:
        ref = np.maximum(ref, 0)
    ref = ref + beta * d0
    assert rel(D.numpy(), ref) < (8e-3 if out == "bf16" else 1e-5)
