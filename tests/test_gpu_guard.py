"""Never read or write outside an operand (matrix.py:5-6,58): every device
operand sits flush against an unmapped guard region -- once at the start of
its mapping (catches reads before the base) and once at the end, exactly
(n-1)*ld+m doubles long (catches reads past the last valid element) -- and
every kernel family and launch plan runs on it.  A stray access faults
(illegal address) instead of silently reading a neighbour's memory; the
results must also equal those of ordinarily allocated operands.  Runs in a
subprocess so a fault cannot poison the test process's CUDA context.
(compute-sanitizer is closed on this GPU pool: this is the stand-in.)"""

import os
import subprocess
import sys
import textwrap

import pytest

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = textwrap.dedent(r"""
    import sys
    sys.path.insert(0, {repo!r})
    import torch
    from cuda.bindings import driver as drv
    from paper_1609_00076_b200 import engine

    torch.zeros(1, device="cuda")
    st = torch.cuda.current_stream().cuda_stream

    def ok(r):
        err = r[0] if isinstance(r, tuple) else r
        assert err == drv.CUresult.CUDA_SUCCESS, err
        return r[1] if isinstance(r, tuple) and len(r) > 1 else None

    prop = drv.CUmemAllocationProp()
    prop.type = drv.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
    prop.location.type = drv.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
    prop.location.id = 0
    gran = ok(drv.cuMemGetAllocationGranularity(
        prop, drv.CUmemAllocationGranularity_flags.CU_MEM_ALLOC_GRANULARITY_MINIMUM))
    keep = []

    def guarded(ndoubles, at_end):
        nbytes = ndoubles * 8
        size = (nbytes + gran - 1) // gran * gran
        va = int(ok(drv.cuMemAddressReserve(size + 2 * gran, 0, 0, 0)))
        h = ok(drv.cuMemCreate(size, prop, 0))
        ok(drv.cuMemMap(va + gran, size, 0, h, 0))
        acc = drv.CUmemAccessDesc()
        acc.location = prop.location
        acc.flags = drv.CUmemAccess_flags.CU_MEM_ACCESS_FLAGS_PROT_READWRITE
        ok(drv.cuMemSetAccess(va + gran, size, [acc], 1))
        keep.append((va, h, size))
        return va + gran + (size - nbytes if at_end else 0)

    def run(m, n, k, lda, ldb, ldc, strips=0, exact=False, at_end=True):
        na, nb, nc = (k - 1) * lda + m, (n - 1) * ldb + k, (n - 1) * ldc + m
        pa, pb, pc = guarded(na, at_end), guarded(nb, at_end), guarded(nc, at_end)
        for p, r, c, ld, seed in ((pa, m, k, lda, 1), (pb, k, n, ldb, 2), (pc, m, n, ldc, 3)):
            engine.fill_random_device(p, r, c, ld, seed, 0, st)
        engine.dgemm_device(m, n, k, pa, lda, pb, ldb, pc, ldc, st, exact=exact, strips=strips,
                            force_tiled=strips > 0)
        torch.cuda.synchronize()
        ref = [torch.full((x,), 0.0, dtype=torch.float64, device="cuda") for x in (na, nb, nc)]
        for t, r, c, ld, seed in ((ref[0], m, k, lda, 1), (ref[1], k, n, ldb, 2), (ref[2], m, n, ldc, 3)):
            engine.fill_random_device(t.data_ptr(), r, c, ld, seed, 0, st)
        engine.dgemm_device(m, n, k, ref[0].data_ptr(), lda, ref[1].data_ptr(), ldb, ref[2].data_ptr(), ldc,
                            st, exact=exact, strips=strips, force_tiled=strips > 0)
        got = torch.empty(nc, dtype=torch.float64, device="cuda")
        ok(drv.cuMemcpyDtoD(got.data_ptr(), pc, nc * 8))
        torch.cuda.synchronize()
        assert torch.equal(got, ref[2]), (m, n, k, lda, ldb, ldc, strips, exact, at_end)

    cases = [
        (1000, 1100, 300, 1000, 300, 1000), (777, 1029, 201, 781, 205, 780), (2048, 2048, 512, 2048, 512, 2048),
        (4093, 4099, 200, 4100, 202, 4096), (4100, 3000, 130, 4101, 131, 4102), (37, 53, 71, 44, 76, 40),
        (1, 700, 300, 3, 301, 2), (700, 1, 300, 701, 303, 703), (6, 3000, 90, 7, 91, 6), (5000, 7, 60, 5001, 61, 5000),
        (16, 5000, 77, 17, 79, 18), (12, 333, 5, 12, 5, 12), (9, 6000, 64, 9, 64, 9),
    ]
    for at_end in (True, False):
        for (m, n, k, lda, ldb, ldc) in cases:
            run(m, n, k, lda, ldb, ldc, at_end=at_end)
            if m > 16 and n > 16:
                for strips in (2, 4, 8, 16, 32, 34, 36, 40) + tuple(range(65, 75)):  # + small-block variants
                    if strips >= 65 and m * n * k > 1e9:
                        continue
                    run(m, n, k, lda, ldb, ldc, strips=strips, at_end=at_end)
            if m * n * k < 2e8:
                run(m, n, k, lda, ldb, ldc, exact=True, at_end=at_end)
    if "--control" in sys.argv:  # negative control: a call one column too wide must fault
        m, n, k = 1000, 1000, 300
        pa, pb, pc = guarded((k - 1) * m + m, True), guarded((n - 1) * k + k, True), guarded((n - 1) * m + m, True)
        try:
            engine.dgemm_device(m, n + 8, k, pa, m, pb, k, pc, m, st)  # reads B and C past the end
            torch.cuda.synchronize()
        except Exception as e:  # CudaError from the library or torch
            print("CONTROL-FAULTED", type(e).__name__)
            sys.exit(0)
        print("CONTROL-NOT-DETECTED")
        sys.exit(1)
    print("GUARD-OK", len(cases))
""")


def test_guard_regions_catch_a_stray_access(tmp_path):
    """Negative control: the guard layout does turn an out-of-bounds access
    into a fault (a call told the matrix is wider than its buffer)."""
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    script = tmp_path / "guard.py"
    script.write_text(SCRIPT.replace("    cases = [", "    cases = [] and [").format(repo=REPO))
    r = subprocess.run([sys.executable, str(script), "--control"], capture_output=True, text=True, timeout=300)
    assert "CONTROL-FAULTED" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]


def test_no_access_outside_operands(tmp_path):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    script = tmp_path / "guard.py"
    script.write_text(SCRIPT.format(repo=REPO))
    r = subprocess.run([sys.executable, str(script)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert "GUARD-OK" in r.stdout
