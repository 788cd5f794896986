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

    python tests/golden/make_golden.py --parts sampled,kat_large

regenerates only the named parts and merges them into the existing
golden.json (parts: base = generator/seed/pack pins, kat = full-GEMM hashes
up to 2048 plus cfg3/cfg4, kat_large = cfg2 2304..8192, sampled = the 64 x 64
sampled grids of cfg2@8192 and cfg5).
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


def sample_grid(m: int, n: int, tile: int = 128, shards: int = 8, count: int = 64):
    """64 row and 64 column indices: the first and last elements, every
    tile-boundary pair (127/128, 255/256, ...) near both ends, the 2-, 4- and
    8-way jc shard boundaries (split_columns: n/G per rank when 128 | n/G),
    the middle, and seeded random fill up to `count`."""
    def pick(size, with_shards):
        idx = {0, 1, 2, 7, 8, 15, 16, 31, 32, 63, 64, size // 2 - 1, size // 2, size - 2, size - 1}
        for t in (1, 2, 3, 4):
            idx.update({t * tile - 1, t * tile, size - t * tile - 1, size - t * tile})
        if with_shards:
            for g in range(1, shards):
                idx.update({g * size // shards - 1, g * size // shards})
        rng = np.random.default_rng(size * 7919 + (1 if with_shards else 0))
        while len(idx) < count:
            idx.add(int(rng.integers(0, size)))
        return sorted(idx)
    return pick(m, False), pick(n, True)


def sampled_elements(name, m, n, k):
    """C_ref(i, j) on the sample grid, each element gemm_naive on the 1 x k
    row of A and the k x 1 column of B plus c_ij (bitwise the full-GEMM
    element: the per-element order is p-ascending).  A's rows come from
    random_values over each column p of A (positions p*m .. p*m+m-1)."""
    rows, cols = sample_grid(m, n)
    sa, sb, sc = (_operand_seed(SEED, r, m, n, k) for r in (1, 2, 3))
    ridx = np.asarray(rows)
    arows = np.empty((len(rows), k))
    for p in range(k):
        arows[:, p] = random_values(sa, m, start=p * m)[ridx]
    vals = []
    for r, i in enumerate(rows):
        arow = Matrix(1, k, 1, np.ascontiguousarray(arows[r]))
        for j in cols:
            bcol = Matrix(k, 1, k, random_values(sb, k, start=j * k))
            cij = Matrix(1, 1, 1, random_values(sc, 1, start=j * m + i))
            vals.append(float(gemm_naive(arow, bcol, cij).data[0]))
    return {"m": m, "n": n, "k": k, "rows": rows, "cols": cols, "values": vals}


def main():
    import argparse

    ap = argparse.ArgumentParser()
    ap.add_argument("--parts", default="base,kat,kat_large,sampled")
    parts = set(ap.parse_args().parts.split(","))
    t0 = time.time()
    path = os.path.join(HERE, "golden.json")
    out: dict = {}
    if parts != {"base", "kat", "kat_large", "sampled"} and os.path.exists(path):
        with open(path) as f:
            out = json.load(f)  # merge the regenerated parts into the committed fixtures
    out.update({"reference": "gemmforge " + gemmforge.__version__, "seed": SEED})
    if "base" not in parts:
        return main_parts(out, parts, path, t0)

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

    return main_parts(out, parts, path, t0)


def main_parts(out, parts, path, t0):
    # -- full-GEMM known answers (sha256 of the valid region) --
    kat = out.get("kat", {})
    full_small = {}
    cases = []
    if "kat" in parts:
        cases += [("cfg1", 512, 512, 512, None)]
        cases += [(f"cfg2_{s}", s, s, s, None) for s in range(256, 2048 + 1, 256) if s != 512]
        cases += [
            ("cfg3a", 4093, 4099, 2047, (4093 + 7, 2047 + 5, 4093 + 3)),
            ("cfg3b", 1, 8192, 8192, (1 + 7, 8192 + 5, 1 + 3)),
            ("cfg3c", 8192, 1, 8192, (8192 + 7, 8192 + 5, 8192 + 3)),
            ("cfg3d", 37, 53, 71, (37 + 7, 71 + 5, 37 + 3)),
            ("cfg4", 16384, 16384, 256, None),
        ]
    if "kat_large" in parts:  # the rest of the cfg2 sweep: every timed size has a bitwise KAT
        cases += [(f"cfg2_{s}", s, s, s, None) for s in range(2304, 8192 + 1, 256)]
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
    if "kat" not in parts:
        return finish(out, parts, path, t0, full_small)

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

    return finish(out, parts, path, t0, full_small)


def finish(out, parts, path, t0, full_small):
    # -- sampled elements of the big shapes: 64 x 64 grids with tile and
    #    shard boundaries (SURVEY 8d oracle coverage) --
    if "sampled" in parts:
        sampled = out.get("sampled", {})
        for name, (m, n, k) in (("cfg2_8192", (8192, 8192, 8192)), ("cfg5", (32768, 32768, 32768))):
            t1 = time.time()
            sampled[name] = sampled_elements(name, m, n, k)
            print(f"sampled {name}: {time.time() - t1:.1f}s", flush=True)
        out["sampled"] = sampled

    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    if full_small:
        np.savez_compressed(os.path.join(HERE, "small_cases.npz"), **full_small)
    print(f"wrote golden fixtures in {time.time() - t0:.1f}s")


if __name__ == "__main__":
    main()
