"""Generate the committed golden fixtures by running the REFERENCE itself.

Run in the build container (where /root/reference exists) after
`oracle/build_ref.sh` has built the unmodified reference package into
oracle/_ref/:

    python tests/golden/make_golden.py

Everything written here comes from the reference's own code path
(gemmforge.matrix.fill_random / random_values, gemmforge.bench._operand_seed
and make_operands, gemmforge.parallel.gemm_goto_parallel with the compiled
backend -- bitwise equal to gemm_naive, reference test_acceptance.py:114-168 --
and gemmforge.kernels.gemm_naive for the sampled elements).  None of it comes
from oracle/, which the fixtures then pin (tests/test_oracle.py).

Output: tests/golden/golden.json (hashes, sampled values, seeds) and
tests/golden/small_cases.npz (full C_ref of the small shapes).
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(REPO, "oracle", "_ref"))

import gemmforge  # noqa: E402  (the reference package)
from gemmforge.backends import available_backends  # noqa: E402
from gemmforge.bench import _operand_seed, make_operands  # noqa: E402
from gemmforge.goto import GotoParams, pack_a, pack_b  # noqa: E402
from gemmforge.kernels import gemm_naive  # noqa: E402
from gemmforge.matrix import (  # noqa: E402
    Matrix,
    alloc_matrix,
    copy_matrix,
    fill_random,
    random_values,
    to_array,
)
from gemmforge.parallel import gemm_goto_parallel, make_plan  # noqa: E402

assert "c" in available_backends(), "build oracle/_ref first (oracle/build_ref.sh)"
T = len(os.sched_getaffinity(0))
SEED = 42


def sha_valid(mat: Matrix) -> str:
    h = hashlib.sha256()
    for j in range(mat.n):
        h.update(np.ascontiguousarray(mat.data[j * mat.ld : j * mat.ld + mat.m]).astype("<f8").tobytes())
    return h.hexdigest()


def reference_gemm(m, n, k, lda=None, ldb=None, ldc=None):
    """C_ref for make_operands(42, m, n, k) via the reference's threaded
    five-loop engine (bitwise gemm_naive).  Padded lds re-fill with the same
    per-role seeds (values are ld-independent)."""
    if lda is None:
        a, b, c = make_operands(SEED, m, n, k)
    else:
        a = fill_random(alloc_matrix(m, k, lda), _operand_seed(SEED, 1, m, n, k))
        b = fill_random(alloc_matrix(k, n, ldb), _operand_seed(SEED, 2, m, n, k))
        c = fill_random(alloc_matrix(m, n, ldc), _operand_seed(SEED, 3, m, n, k))
    p = GotoParams()
    if -(-m // p.mc) >= T:
        plan = make_plan("ic", T, m, p.mc)
    else:
        plan = make_plan("jr", T, n, p.nr)
    gemm_goto_parallel(a, b, c, p, plan)
    return a, b, c


def main():
    t0 = time.time()
    out: dict = {"reference": "gemmforge " + gemmforge.__version__, "seed": SEED}

    # -- generator pins (matrix.py:184-207; reference tests/test_matrix.py) --
    out["random_values"] = {
        "seed42_first8": random_values(42, 8).tolist(),
        "seed0_first3": random_values(0, 3).tolist(),
        "seed_max_first3": random_values((1 << 64) - 1, 3).tolist(),
        "seed12345678901234567_first3": random_values(12345678901234567, 3).tolist(),
        "seed7_start123457_count16": random_values(7, 16, start=123457).tolist(),
        "seed9_3x5_ld7": to_array(fill_random(alloc_matrix(3, 5, 7), 9)).T.ravel().tolist(),
    }
    # -- operand seeds (bench.py:89-98) --
    shapes = {
        "cfg1": (512, 512, 512),
        "cfg3a": (4093, 4099, 2047),
        "cfg3b": (1, 8192, 8192),
        "cfg3c": (8192, 1, 8192),
        "cfg3d": (37, 53, 71),
        "cfg4": (16384, 16384, 256),
        "cfg5": (32768, 32768, 32768),
        "cfg2_8192": (8192, 8192, 8192),
    }
    out["operand_seeds"] = {
        name: [hex(_operand_seed(SEED, r, *s)) for r in (1, 2, 3)] for name, s in shapes.items()
    }

    # -- packing layouts (goto.py:116-135) --
    a = fill_random(alloc_matrix(7, 5, 9), 201)
    b = fill_random(alloc_matrix(5, 7, 6), 211)
    out["pack"] = {
        "a_7x5_ld9_seed201_mr3": pack_a(a, 3).buffer.tolist(),
        "b_5x7_ld6_seed211_nr3": pack_b(b, 3).buffer.tolist(),
    }

    # -- full-GEMM known answers (sha256 of the valid region) --
    kat = {}
    full_small = {}
    cases = [("cfg1", 512, 512, 512, None)]
    cases += [(f"cfg2_{s}", s, s, s, None) for s in range(256, 2048 + 1, 256) if s != 512]
    cases += [
        ("cfg3a", 4093, 4099, 2047, (4093 + 7, 2047 + 5, 4093 + 3)),
        ("cfg3b", 1, 8192, 8192, (1 + 7, 8192 + 5, 1 + 3)),
        ("cfg3c", 8192, 1, 8192, (8192 + 7, 8192 + 5, 8192 + 3)),
        ("cfg3d", 37, 53, 71, (37 + 7, 71 + 5, 37 + 3)),
        ("cfg4", 16384, 16384, 256, None),
    ]
    for name, m, n, k, lds in cases:
        t1 = time.time()
        if lds is None:
            a, b, c = reference_gemm(m, n, k)
        else:
            a, b, c = reference_gemm(m, n, k, *lds)
        kat[name] = {"m": m, "n": n, "k": k, "lds": list(lds) if lds else [m, k, m],
                     "sha256": sha_valid(c), "c00": float(c.data[0]),
                     "c_last": float(c.data[(n - 1) * c.ld + m - 1])}
        if m * n <= 4096:
            full_small[name] = to_array(c)
        print(f"{name}: {time.time() - t1:.1f}s", flush=True)
    out["kat"] = kat

    # -- small problems: registry gate and CLI verify shapes (registry.py:46-51,
    #    127-137; cli.py:66), full C_ref arrays --
    def random_problem(m, n, k, seed):
        a = fill_random(alloc_matrix(m, k), seed)
        b = fill_random(alloc_matrix(k, n), seed + 1)
        c = fill_random(alloc_matrix(m, n), seed + 2)
        return a, b, c

    for m, n, k, s in ((5, 4, 3, 21), (8, 8, 8, 22), (9, 7, 11, 23)):
        a, b, c = random_problem(m, n, k, 2000 + s)
        full_small[f"gate_{m}_{n}_{k}_seed{2000 + s}"] = to_array(gemm_naive(a, b, copy_matrix(c)))
    for m, n, k in ((8, 8, 8), (16, 16, 16), (31, 33, 32), (64, 64, 64), (97, 89, 83)):
        a, b, c = make_operands(SEED, m, n, k)
        full_small[f"verify_{m}_{n}_{k}"] = to_array(gemm_naive(a, b, c))

    # -- sampled elements of the big shapes (gemm_naive on a 1 x k row of A and
    #    a k x 1 column of B plus c_ij: bitwise the full-GEMM element) --
    sampled = {}
    for name, (m, n, k) in (("cfg2_8192", (8192, 8192, 8192)), ("cfg5", (32768, 32768, 32768))):
        rows = [0, 1, 127, 128, m // 2 + 3, m - 2, m - 1]
        cols = [0, 1, 63, 64, n // 3, n - 1]
        sa, sb, sc = (_operand_seed(SEED, r, m, n, k) for r in (1, 2, 3))
        vals = []
        for i in rows:
            arow = Matrix(1, k, 1, np.ascontiguousarray(
                [random_values(sa, 1, start=p * m + i)[0] for p in range(k)]))
            for j in cols:
                bcol = Matrix(k, 1, k, random_values(sb, k, start=j * k))
                cij = Matrix(1, 1, 1, random_values(sc, 1, start=j * m + i))
                vals.append(float(gemm_naive(arow, bcol, cij).data[0]))
        sampled[name] = {"m": m, "n": n, "k": k, "rows": rows, "cols": cols, "values": vals}
        print(f"sampled {name}: done", flush=True)
    out["sampled"] = sampled

    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(out, f, indent=1)
    np.savez_compressed(os.path.join(HERE, "small_cases.npz"), **full_small)
    print(f"wrote golden fixtures in {time.time() - t0:.1f}s")


if __name__ == "__main__":
    main()
