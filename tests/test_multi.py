"""Host logic of the jc-sharded multi-GPU driver (paper_1609_00076_b200/multi.py)
on CPU: planning rules, and a real world_size-2 gloo run whose A broadcast
and chunk ordering are the product code, with the oracle injected as the
per-rank compute (tests may call the oracle; the product never does)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1609_00076_b200.multi import (
    ShardedDgemm,
    a_span,
    k_chunks,
    make_shard_plan,
    split_columns,
)


def test_split_columns_balanced_and_aligned():
    assert split_columns(32768, 8) == tuple((i * 4096, (i + 1) * 4096) for i in range(8))
    assert split_columns(1000, 3) == ((0, 384), (384, 768), (768, 1000))
    assert split_columns(100, 4) == ((0, 100), (100, 100), (100, 100), (100, 100))
    assert split_columns(0, 2) == ((0, 0), (0, 0))
    for n, w in ((65536, 8), (8192, 3), (129, 2), (4099, 4)):
        parts = split_columns(n, w)
        assert parts[0][0] == 0 and parts[-1][1] == n
        assert all(lo <= hi for lo, hi in parts)
        assert all(parts[i][1] == parts[i + 1][0] for i in range(w - 1))
    with pytest.raises(ValueError):
        split_columns(-1, 2)
    with pytest.raises(ValueError):
        split_columns(4, 0)


def test_k_chunks_multiple_of_16_and_cover():
    assert k_chunks(100, 40) == ((0, 48), (48, 96), (96, 100))
    assert k_chunks(5, 1) == ((0, 5),)
    ch = k_chunks(32768, 2048)
    assert len(ch) == 16 and ch[-1] == (30720, 32768)
    with pytest.raises(ValueError):
        k_chunks(0, 16)


def test_a_span_never_reads_past_last_valid_element():
    m, lda, k = 5, 8, 6
    lo, hi = a_span(lda, m, 4, 6)
    assert (lo, hi) == (32, 45)
    assert hi == (k - 1) * lda + m


def test_plan_world1_single_chunk():
    p = make_shard_plan(64, 64, 1000, 1)
    assert p.chunks == ((0, 1000),) and p.columns == ((0, 64),)
    with pytest.raises(ValueError):
        make_shard_plan(0, 1, 1, 1)
    with pytest.raises(ValueError):
        make_shard_plan(1, 1, 1, 2, root=2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, shape, lds, k_chunk, overlap, out_q, host=False):
    import oracle

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m, n, k = shape
        lda, ldb, ldc = lds
        a, b, c = oracle.make_padded_operands(42, m, n, k, lda, ldb, ldc, canary=-9.0)
        plan = make_shard_plan(m, n, k, world, root=0, k_chunk=k_chunk)
        j0, j1 = plan.local(rank)
        A = torch.from_numpy(a.copy()) if rank == 0 else torch.full_like(torch.from_numpy(a), -1.0)
        B_local = torch.from_numpy(b[j0 * ldb:j1 * ldb].copy())
        C_local = torch.from_numpy(c[j0 * ldc:j1 * ldc].copy())
        calls = []

        def compute(m_, nloc, kc, A_, lda_, B_, ldb_, C_, ldc_):
            calls.append(kc)
            oracle.naive(m_, nloc, kc, A_.numpy(), lda_, B_.numpy(), ldb_, C_.numpy(), ldc_)

        drv = ShardedDgemm(plan, rank, compute=compute, overlap=overlap)
        if host:  # step_host: operands start in host buffers, device-side buffers hold junk
            hA, hB, hC = A.clone(), B_local.clone(), C_local.clone()
            A.fill_(-1.0)
            B_local.fill_(-2.0)
            C_local.fill_(-3.0)
            out = drv.step_host(hA, A, lda, hB, B_local, ldb, hC, C_local, ldc)
            assert out is hC
            C_local = hC
        else:
            drv.step(A, lda, B_local, ldb, C_local, ldc)
        # valid region of A arrived; padding rows were never sent
        got_a = oracle.valid_region(A.numpy(), m, k, lda)
        out_q.put((rank, j0, j1, C_local.numpy().copy(), calls,
                   np.array_equal(got_a, oracle.valid_region(a, m, k, lda))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("shape,lds,k_chunk,overlap,host", [
    ((37, 300, 71), (44, 76, 40), 32, True, False),
    ((16, 129, 50), (16, 50, 16), 16, True, False),   # few-row path: one k chunk (only the tiled family chunks k)
    ((20, 129, 50), (20, 50, 21), 16, True, False),
    ((37, 300, 71), (44, 76, 40), 32, False, False),
    ((37, 300, 71), (44, 76, 40), 32, True, True),    # step_host: uploads, chunked broadcast, download
    ((37, 300, 71), (44, 76, 40), 32, False, True),
])
def test_gloo_world2_sharded_step_bitwise_equals_oracle(shape, lds, k_chunk, overlap, host):
    import oracle

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, shape, lds, k_chunk, overlap, q, host))
             for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    m, n, k = shape
    lda, ldb, ldc = lds
    a, b, c = oracle.make_padded_operands(42, m, n, k, lda, ldb, ldc, canary=-9.0)
    want = oracle.naive(m, n, k, a, lda, b, ldb, c.copy(), ldc)
    from paper_1609_00076_b200 import _capi, engine

    nchunks = len(k_chunks(k, k_chunk)) if overlap and engine.path(m, n) == _capi.PATH_TILED else 1
    for rank, j0, j1, cl, calls, a_ok in sorted(results, key=lambda t: t[0]):
        assert a_ok, f"rank {rank} did not receive A"
        if j1 > j0:
            assert len(calls) == nchunks and sum(calls) == k
            assert np.array_equal(cl[: (j1 - j0) * ldc], want[j0 * ldc: j1 * ldc]), rank
