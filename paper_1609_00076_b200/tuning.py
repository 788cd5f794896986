"""Tile-parameter grid tuner: the GPU restatement of the reference's
``tune`` (pkg/src/gemmforge/bench.py:238-311).

The reference grid-searches its blocking parameters (mr, nr, mc, kc, nc) at
one probe size: each grid point is validated first (parameter invariants,
blocks larger than the probe are skipped with a warning), timed best-of-reps,
verified once against the oracle, and the best rate wins, exact ties going
to the smaller packed footprint mc*kc + kc*nc, then to the lexicographically
smaller parameters.

Here the blocking parameters are the CTA block bm x bn, the K-slab depth bk
and the shared-memory ring depth ``stages`` -- what the reference's mc / nc
/ kc and packing buffers become on the GPU.  They are compile-time template
parameters, so the grid is searched over the instantiations the library
carries (``my_dgemm_plan_geometry``): the persistent kernel's launch plans
(128x128 tiles, 128x64 / 128x32 / 64x32 / 16x128 units, stream-K) and the
small-block kernel's variants.  A grid point that no compiled instantiation
has is skipped with a warning (the analogue of ``param_violations``), as is
one whose blocks exceed the probe size.  Each surviving point runs on
device-resident operands from the reference generator, is timed best-of-reps
with CUDA events, and is verified once against the exact kernel (the bitwise
twin of the reference's oracle) with the reference tolerance
(kernels.py:31-38); a failure raises VerificationError with the reference's
failure line.  Ties prefer the smaller shared-memory footprint
stages * (bk*bm + bn*bk) doubles, then the smaller key.  Every plan computes
bitwise the same C, so tuning changes speed, never results.
"""

from __future__ import annotations

import ctypes
import itertools
import sys
from dataclasses import dataclass, field

from . import _capi
from . import engine

AXES = ("bm", "bn", "bk", "stages")
PLANS = (1, 2, 4, 8, 16, 32, 34, 36, 40) + tuple(range(65, 75))
REF_SEED = 42  # the reference's default Config.seed (config.py)


@dataclass(frozen=True)
class TilePoint:
    bm: int
    bn: int
    bk: int
    stages: int
    plan: int

    @property
    def key(self) -> tuple[int, int, int, int]:
        return (self.bm, self.bn, self.bk, self.stages)

    @property
    def footprint(self) -> int:
        """Shared-memory ring footprint in doubles (the reference's mc*kc + kc*nc)."""
        return self.stages * (self.bk * self.bm + self.bn * self.bk)


@dataclass
class TileTuneResult:
    best: TilePoint
    rate: float  # GFLOP/s at the probe size
    table: dict = field(default_factory=dict)  # TilePoint -> GFLOP/s
    probe_size: int = 0
    skipped: list = field(default_factory=list)  # (point, reason)


def plan_geometry(plan: int, k: int, vec2: bool = True) -> TilePoint | None:
    """The compiled blocking parameters of a launch plan at depth k."""
    lib = _capi.load()
    v = [ctypes.c_int() for _ in range(4)]
    if lib.my_dgemm_plan_geometry(plan, k, 1 if vec2 else 0, *[ctypes.byref(x) for x in v]) != 0:
        return None
    return TilePoint(v[0].value, v[1].value, v[2].value, v[3].value, plan)


def describe_plan(m: int, n: int, k: int, lda: int | None = None, ldb: int | None = None, ldc: int | None = None,
                  plan: int = 0) -> dict:
    """The tiled path's launch plan for a shape, from the planner itself
    (my_dgemm_plan_describe: host code, nothing is launched, no GPU needed --
    without a device it plans for 148 SMs).  The reference's make_plan
    (pkg/src/gemmforge/parallel.py:60-105) as data: `kind` is "units",
    "stream-K", "K-split" or "small"; `split` / `sk_split` the units per tile
    (1 = full 128x128 tiles), `sk_dp_rounds` the whole-tile rounds ahead of a
    full-tile stream-K phase, `q` the whole-tile rounds (or tiles) of the main
    launch, `edge` the edge plan, `small` the small-block variant, `model_us`
    the planner's cost of its persistent-kernel choice, `small_us` the
    small-block kernel's cheapest variant by its own model (-1 when not
    evaluated).  plan: 0 the heuristic,
    -1 the heuristic kept to plan-invariant plans, else a pinned plan id."""
    lib = _capi.load()
    buf = ctypes.create_string_buffer(512)
    st = lib.my_dgemm_plan_describe(m, n, k, lda or m, ldb or k, ldc or m, plan, buf, len(buf))
    if st != 0:
        raise ValueError(f"my_dgemm_plan_describe({m}, {n}, {k}) failed with status {st}")
    text = buf.value.decode()
    out: dict = {"text": text}
    for tok in text.split():
        if "=" in tok:
            key, val = tok.split("=", 1)
            out[key] = float(val) if key.endswith("_us") else (val if "x" in val else int(val))
        else:
            out["kind"] = tok
    return out


def compiled_points(k: int, vec2: bool = True) -> list[TilePoint]:
    """Every launch plan's blocking parameters at depth k (one point per plan;
    stream-K plans share their unit shape's geometry)."""
    return [p for p in (plan_geometry(plan, k, vec2) for plan in PLANS) if p is not None]


def grid_points(grid: dict, k: int, vec2: bool = True) -> tuple[list[TilePoint], list[tuple[tuple, str]]]:
    """Expand `grid` (axis -> candidate values; a missing axis accepts every
    compiled value) into the compiled plans that realise each point, and the
    points no instantiation has (skipped, with the reason)."""
    for key in grid:
        if key not in AXES:
            raise ValueError(f"unknown tile axis {key!r}; choose from {', '.join(AXES)}")
    have = compiled_points(k, vec2)
    axes = [sorted(set(grid[a])) if a in grid else sorted({getattr(p, a) for p in have}) for a in AXES]
    chosen, skipped = [], []
    for combo in itertools.product(*axes):
        match = [p for p in have if p.key == combo]
        if not match:
            if all(a in grid for a in AXES):  # an explicit point the library does not carry
                skipped.append((combo, "no compiled instantiation with these tile parameters"))
            continue
        chosen.extend(match)
    return chosen, skipped


def _beats(rate: float, pt: TilePoint, best_rate: float, best: TilePoint | None) -> bool:
    if best is None or rate > best_rate:
        return True
    if rate < best_rate:
        return False
    return (pt.footprint, pt.key, pt.plan) < (best.footprint, best.key, best.plan)


def tune_grid(grid: dict, probe_size: int, reps: int = 3, log=None, apply: bool = True,
              shape: tuple[int, int, int] | None = None) -> TileTuneResult:
    """Grid-search the tile parameters at one probe size (m = n = k =
    probe_size, or `shape`); see the module docstring.  apply=True pins the
    winner for later calls of that shape (my_dgemm_tune_set)."""
    import torch

    if probe_size < 1:
        raise ValueError(f"probe_size must be positive, got {probe_size}")
    log = sys.stderr if log is None else log
    m, n, k = shape if shape is not None else (probe_size, probe_size, probe_size)
    points, skipped = grid_points(grid, k)
    st = torch.cuda.current_stream().cuda_stream
    dev = lambda rows, cols: torch.empty(rows * cols, dtype=torch.float64, device="cuda")  # noqa: E731
    a, b, c0 = dev(m, k), dev(k, n), dev(m, n)
    for role, (buf, rows, cols) in enumerate(((a, m, k), (b, k, n), (c0, m, n)), start=1):
        engine.fill_random_device(buf.data_ptr(), rows, cols, rows, engine.operand_seed(REF_SEED, role, m, n, k), 0,
                                  st)
    want = c0.clone()
    engine.dgemm_device(m, n, k, a.data_ptr(), m, b.data_ptr(), k, want.data_ptr(), m, st, exact=True)
    # reference tolerance (kernels.py:31-38): 2^-50 * k * max|A| * max|B|
    tol = 2.0 ** -50 * k * float(a.abs().max()) * float(b.abs().max())
    table, best, best_rate = {}, None, -1.0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for pt in points:
        if pt.bm > m or pt.bn > n or pt.bk > k:
            reason = f"block sizes exceed probe size {probe_size}"
            print(f"tune: skipping bm={pt.bm} bn={pt.bn} bk={pt.bk} stages={pt.stages} (plan {pt.plan}): {reason}",
                  file=log)
            skipped.append((pt.key, reason))
            continue
        got = c0.clone()
        engine.dgemm_device(m, n, k, a.data_ptr(), m, b.data_ptr(), k, got.data_ptr(), m, st, strips=pt.plan,
                            force_tiled=True)
        engine.verify_device(m, n, k, got.data_ptr(), m, want.data_ptr(), m, tol, algorithm=f"b200 plan {pt.plan}")
        t_best = float("inf")
        for _ in range(max(1, reps)):
            c = c0.clone()
            e0.record()
            engine.dgemm_device(m, n, k, a.data_ptr(), m, b.data_ptr(), k, c.data_ptr(), m, st, strips=pt.plan,
                                force_tiled=True)
            e1.record()
            torch.cuda.synchronize()
            t_best = min(t_best, e0.elapsed_time(e1) * 1e-3)
        rate = 2.0 * m * n * k / t_best / 1e9
        table[pt] = rate
        if _beats(rate, pt, best_rate, best):
            best, best_rate = pt, rate
    for combo, reason in skipped:
        if reason.startswith("no compiled"):
            print(f"tune: skipping bm={combo[0]} bn={combo[1]} bk={combo[2]} stages={combo[3]}: {reason}", file=log)
    if best is None:
        raise ValueError("no valid grid points to tune over")
    if apply:
        _capi.check(_capi.load().my_dgemm_tune_set(m, n, k, m, k, best.plan))
    return TileTuneResult(best, best_rate, table, probe_size, skipped)
