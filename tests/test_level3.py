"""GEMM-based level-3 BLAS (my_dsyrk / my_dtrmm / my_dtrsm; SURVEY.md 8f rank 4,
"poorman's BLAS").  CPU: reference-BLAS argument checks and
quick returns through the C ABI (no GPU needed: validation precedes any device
work).  GPU: every side / uplo / trans / diag case against numpy fp64, with
padded leading dimensions, canaries in the padding and in the untouched
triangle."""
import itertools

import numpy as np
import pytest

from paper_1609_00076_b200 import _capi, engine

EPS = 2.0 ** -52


@pytest.fixture(scope="module")
def lib():
    return _capi.load()


def test_level3_argument_checks(lib):
    a = np.zeros(64)
    p = a.ctypes.data
    D = _capi.DEVICE_PTRS
    cases = [
        (lib.my_dtrsm, (b"X", b"L", b"N", b"N", 4, 4, 1.0, p, 4, p, 4, D, None), -1, "side"),
        (lib.my_dtrsm, (b"L", b"Q", b"N", b"N", 4, 4, 1.0, p, 4, p, 4, D, None), -2, "uplo"),
        (lib.my_dtrmm, (b"L", b"U", b"Z", b"N", 4, 4, 1.0, p, 4, p, 4, D, None), -3, "transa"),
        (lib.my_dtrmm, (b"L", b"U", b"N", b"Z", 4, 4, 1.0, p, 4, p, 4, D, None), -4, "diag"),
        (lib.my_dtrsm, (b"L", b"U", b"N", b"N", -1, 4, 1.0, p, 4, p, 4, D, None), -5, "m must"),
        (lib.my_dtrsm, (b"L", b"U", b"N", b"N", 4, -1, 1.0, p, 4, p, 4, D, None), -6, "n must"),
        (lib.my_dtrsm, (b"L", b"U", b"N", b"N", 4, 3, 1.0, p, 3, p, 4, D, None), -9, "lda=3"),
        (lib.my_dtrsm, (b"R", b"U", b"N", b"N", 4, 6, 1.0, p, 5, p, 4, D, None), -9, "lda=5"),
        (lib.my_dtrmm, (b"R", b"U", b"N", b"N", 4, 3, 1.0, p, 3, p, 3, D, None), -11, "ldb=3"),
        (lib.my_dtrmm, (b"R", b"U", b"N", b"N", 4, 3, 1.0, p, 3, p, 4, 0, None), -12, "device pointers"),
        (lib.my_dsyrk, (b"A", b"N", 4, 4, 1.0, p, 4, 1.0, p, 4, D, None), -1, "uplo"),
        (lib.my_dsyrk, (b"U", b"X", 4, 4, 1.0, p, 4, 1.0, p, 4, D, None), -2, "trans"),
        (lib.my_dsyrk, (b"U", b"N", -2, 4, 1.0, p, 4, 1.0, p, 4, D, None), -3, "n must"),
        (lib.my_dsyrk, (b"U", b"N", 4, -2, 1.0, p, 4, 1.0, p, 4, D, None), -4, "k must"),
        (lib.my_dsyrk, (b"U", b"T", 4, 6, 1.0, p, 4, 1.0, p, 4, D, None), -7, "lda=4"),
        (lib.my_dsyrk, (b"U", b"N", 4, 6, 1.0, p, 4, 1.0, p, 3, D, None), -10, "ldc=3"),
        (lib.my_dsyrk, (b"U", b"N", 4, 6, 1.0, p, 4, 1.0, p, 4, 0, None), -11, "device pointers"),
    ]
    for fn, args, want, msg in cases:
        assert fn(*args) == want, (args, want)
        assert msg in _capi.last_error(), (args, _capi.last_error())
    assert not a.any()  # rejected calls touch nothing
    # quick returns: empty problems, and syrk with alpha == 0 / k == 0 and beta == 1
    assert lib.my_dtrsm(b"L", b"U", b"N", b"N", 0, 4, 1.0, None, 1, None, 1, D, None) == 0
    assert lib.my_dtrmm(b"R", b"L", b"T", b"U", 5, 0, 1.0, None, 1, None, 5, D, None) == 0
    assert lib.my_dsyrk(b"L", b"N", 0, 3, 1.0, None, 1, 0.5, None, 1, D, None) == 0
    assert lib.my_dsyrk(b"L", b"N", 5, 0, 1.0, None, 5, 1.0, p, 5, D, None) == 0
    assert lib.my_dsyrk(b"L", b"N", 5, 3, 0.0, None, 5, 1.0, p, 5, D, None) == 0


def _tri_matrix(rng, na, lda, uplo, diag):
    """Well-conditioned triangular A (n x n in an lda-padded buffer): off-diagonal
    uniform [-1, 1) / sqrt(n), diagonal 1 + |u| (ignored when diag == 'U'),
    garbage in the other triangle and NaN in the padding rows, which the
    routines must not read."""
    full = rng.uniform(-1, 1, (na, na)) / np.sqrt(na)
    np.fill_diagonal(full, 1.0 + np.abs(rng.uniform(-1, 1, na)))
    tri = np.tril(full) if uplo == "L" else np.triu(full)
    stored = np.where(tri != 0, tri, 1e30)  # the other triangle holds junk
    if diag == "U":
        np.fill_diagonal(stored, 7e29)
        np.fill_diagonal(tri, 1.0)
    buf = np.full((na, lda), np.nan)  # column-major: buf[col, row]
    buf[:, :na] = stored.T
    return tri, buf


def _op(t, trans):
    return t.T if trans == "T" else t


@pytest.mark.gpu
@pytest.mark.parametrize("side,uplo,trans,diag", list(itertools.product("LR", "LU", "NT", "NU")))
@pytest.mark.parametrize("m,n", [(37, 29), (600, 333), (1100, 70)])
def test_trmm_trsm_all_cases_vs_numpy(side, uplo, trans, diag, m, n):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    rng = np.random.default_rng(hash((side, uplo, trans, diag, m, n)) & 0xFFFF)
    na = m if side == "L" else n
    lda, ldb = na + 3, m + 5
    tri, abuf = _tri_matrix(rng, na, lda, uplo, diag)
    B = rng.uniform(-1, 1, (m, n))
    bbuf = np.full((n, ldb), -777.25)
    bbuf[:, :m] = B.T
    dA = torch.from_numpy(abuf.ravel()).cuda()
    opA = _op(tri, trans)
    alpha = -1.5
    # multiply
    dB = torch.from_numpy(bbuf.ravel().copy()).cuda()
    engine.dtrmm(side, uplo, trans, diag, m, n, alpha, dA, lda, dB, ldb)
    torch.cuda.synchronize()
    got = dB.cpu().numpy().reshape(n, ldb)
    want = alpha * (opA @ B if side == "L" else B @ opA)
    bound = 4 * na * EPS * np.abs(alpha) * (np.abs(opA) @ np.abs(B) if side == "L" else np.abs(B) @ np.abs(opA)).max()
    assert np.abs(got[:, :m].T - want).max() <= bound
    assert np.all(got[:, m:] == -777.25)
    # solve: X with op(A) X = alpha B (left) or X op(A) = alpha B (right)
    dB = torch.from_numpy(bbuf.ravel().copy()).cuda()
    engine.dtrsm(side, uplo, trans, diag, m, n, alpha, dA, lda, dB, ldb)
    torch.cuda.synchronize()
    got = dB.cpu().numpy().reshape(n, ldb)
    X = got[:, :m].T
    assert np.all(np.isfinite(X))
    resid = (opA @ X if side == "L" else X @ opA) - alpha * B
    scale = (np.abs(opA) @ np.abs(X) if side == "L" else np.abs(X) @ np.abs(opA)).max()
    assert np.abs(resid).max() <= 8 * na * EPS * scale, np.abs(resid).max() / (na * EPS * scale)
    assert np.all(got[:, m:] == -777.25)


@pytest.mark.gpu
@pytest.mark.parametrize("uplo,trans", list(itertools.product("LU", "NT")))
@pytest.mark.parametrize("n,k,alpha,beta", [(45, 33, 1.0, 1.0), (700, 300, -0.5, 2.0), (1300, 129, 2.0, 0.0)])
def test_syrk_vs_numpy(uplo, trans, n, k, alpha, beta):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    rng = np.random.default_rng(n * 7 + k)
    rows, cols = (k, n) if trans == "T" else (n, k)
    lda, ldc = rows + 2, n + 3
    A = rng.uniform(-1, 1, (rows, cols))
    abuf = np.full((cols, lda), np.nan)
    abuf[:, :rows] = A.T
    C = rng.uniform(-1, 1, (n, n))
    if beta == 0.0:
        C[:] = np.nan  # beta == 0: C is not read
    cbuf = np.full((n, ldc), -777.25)
    cbuf[:, :n] = C.T
    dA, dC = torch.from_numpy(abuf.ravel()).cuda(), torch.from_numpy(cbuf.ravel().copy()).cuda()
    engine.dsyrk(uplo, trans, n, k, alpha, dA, lda, beta, dC, ldc)
    torch.cuda.synchronize()
    got = dC.cpu().numpy().reshape(n, ldc)[:, :n].T
    opA = A.T if trans == "T" else A
    want = alpha * (opA @ opA.T) + (0.0 if beta == 0.0 else beta * C)
    mask = np.tril(np.ones((n, n), bool)) if uplo == "L" else np.triu(np.ones((n, n), bool))
    cmax = 0.0 if beta == 0.0 else np.abs(C).max()
    bound = 4 * k * EPS * (abs(alpha) * (np.abs(opA) @ np.abs(opA.T)).max() + abs(beta) * cmax)
    assert np.abs(got[mask] - want[mask]).max() <= bound
    other = got[~mask]
    assert np.all(np.isnan(other)) if beta == 0.0 else np.array_equal(other, C[~mask])
    assert np.all(dC.cpu().numpy().reshape(n, ldc)[:, n:] == -777.25)


def _tri_only_product(opA, B, side, lower):
    """op(A) B (left) or B op(A) (right) summing only the triangle's products:
    products outside the triangle are dropped, not multiplied by zero, as
    reference BLAS never reads the other triangle (0 * Inf would be NaN)."""
    na = opA.shape[0]
    mask = np.tril(np.ones((na, na), bool)) if lower else np.triu(np.ones((na, na), bool))
    with np.errstate(invalid="ignore", over="ignore"):
        if side == "L":  # W[r, j] = sum_c opA[r, c] B[c, j]
            prod = opA[:, :, None] * B[None, :, :]
            return np.where(mask[:, :, None], prod, 0.0).sum(axis=1)
        prod = B[:, :, None] * opA[None, :, :]  # W[r, cc] = sum_c B[r, c] opA[c, cc]
        return np.where(mask[None, :, :], prod, 0.0).sum(axis=1)


@pytest.mark.gpu
@pytest.mark.parametrize("side,uplo,trans", list(itertools.product("LR", "LU", "NT")))
def test_trmm_nonfinite_b_reads_triangle_only(side, uplo, trans):
    """Inf / -Inf / NaN in B: the dense 512 diagonal-block
    multiply must not turn 0 * Inf from the unreferenced triangle into NaN.
    Result against a triangle-only evaluation: finite entries within the
    bound, the non-finite pattern (which vectors are Inf / NaN, and the sign
    of each Inf) identical."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    m, n = (600, 24) if side == "L" else (24, 600)  # the triangle's order > 256: the dense-block path
    rng = np.random.default_rng(17)
    na = m if side == "L" else n
    lda, ldb = na + 1, m + 2
    tri, abuf = _tri_matrix(rng, na, lda, uplo, "N")
    B = rng.uniform(-1, 1, (m, n))
    if side == "L":  # one non-finite per column vector, in different 512-blocks' reach
        B[5, 3], B[300, 7], B[550, 11] = np.inf, -np.inf, np.nan
        B[599, 20] = np.inf
    else:
        B[3, 5], B[7, 300], B[11, 550] = np.inf, -np.inf, np.nan
        B[20, 599] = np.inf
    bbuf = np.full((n, ldb), -777.25)
    bbuf[:, :m] = B.T
    dA = torch.from_numpy(abuf.ravel()).cuda()
    dB = torch.from_numpy(bbuf.ravel().copy()).cuda()
    alpha = -1.5
    engine.dtrmm(side, uplo, trans, "N", m, n, alpha, dA, lda, dB, ldb)
    torch.cuda.synchronize()
    got = dB.cpu().numpy().reshape(n, ldb)[:, :m].T
    opA = _op(tri, trans)
    lower = (uplo == "L") != (trans == "T")
    want = _tri_only_product(opA, alpha * B, side, lower)
    assert np.array_equal(np.isnan(got), np.isnan(want))
    assert np.array_equal(np.isposinf(got), np.isposinf(want))
    assert np.array_equal(np.isneginf(got), np.isneginf(want))
    fin = np.isfinite(want)
    assert fin.sum() > 0.5 * fin.size and (~fin).sum() > 0
    Bf = np.where(np.isfinite(B), B, 0.0)
    bound = 4 * na * EPS * 1.5 * (np.abs(opA) @ np.abs(Bf) if side == "L" else np.abs(Bf) @ np.abs(opA)).max()
    assert np.abs(got[fin] - want[fin]).max() <= bound
    assert np.all(dB.cpu().numpy().reshape(n, ldb)[:, m:] == -777.25)
