"""The copy-engine chain exchange of A (paper_1609_00076_b200/peer.py) on CPU.

The chain protocol -- who waits on which flag for which step, who copies
which chunk from whom, who writes which neighbour's flag -- is the product
code (PeerChain, ShardedDgemm.attach_chain).  Only its operations are faked:
each rank's A buffer and flags live in POSIX shared memory, the processes
attach their neighbours' segments (the names exchanged over gloo, as
connect_chain exchanges CUDA IPC handles), waits spin on the flag, writes
store it, copies are memcpys, and the per-rank compute is the oracle.  The
ranks run as real concurrent processes, so a missing or misplaced wait shows
up as a wrong A (a stale or half-copied chunk) or a hang (timeout)."""

import os
import socket
import time
from multiprocessing import shared_memory

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1609_00076_b200.multi import ShardedDgemm, make_shard_plan
from paper_1609_00076_b200.peer import ChainLinks, PeerChain, chain_position


def test_chain_position_is_a_line_from_the_root():
    assert [chain_position(r, 2, 4) for r in range(4)] == [2, 3, 0, 1]
    with pytest.raises(ValueError):
        chain_position(0, 4, 4)


class _Recorder:
    """Records the queued operations of one rank (no execution)."""

    def __init__(self):
        self.log = []

    def record(self, stream):
        self.log.append(("record", stream))
        return len(self.log)

    def wait_event(self, stream, ev):
        self.log.append(("wait_event", stream, ev))

    def wait_geq(self, stream, addr, value):
        self.log.append(("wait", stream, addr, value))

    def write(self, stream, addr, value):
        self.log.append(("write", stream, addr, value))

    def copy(self, stream, dst, src, n):
        self.log.append(("copy", stream, dst, src, n))


def test_middle_rank_operation_order():
    """A middle rank: per chunk wait own ready -> pull from pred -> free pred
    -> signal succ; end of step: wait own freed for every chunk."""
    ops = _Recorder()
    links = ChainLinks(a_local=1000, flags_local=500, a_pred=9000, flags_pred=700, flags_succ=900)
    ch = PeerChain(links, [(0, 10), (16, 20)], position=1, world=3, ops=ops, copy_stream="cp")
    evs = ch.issue("cs")
    ch.finish("cs")
    assert ops.log == [
        ("record", "cs"), ("wait_event", "cp", 1),
        ("wait", "cp", 500, 1), ("copy", "cp", 1000, 9000, 80), ("write", "cp", 708, 1), ("record", "cp"),
        ("write", "cp", 900, 1),
        ("wait", "cp", 504, 1), ("copy", "cp", 1128, 9128, 32), ("write", "cp", 712, 1), ("record", "cp"),
        ("write", "cp", 904, 1),
        ("wait", "cs", 508, 1), ("wait", "cs", 512, 1),
    ]
    assert evs == [6, 11]
    ch.issue("cs")
    assert ch.step == 2 and ops.log[-1] == ("write", "cp", 904, 2)


def test_root_and_last_rank_roles():
    ops = _Recorder()
    root = PeerChain(ChainLinks(0, 64, None, None, 128), [(0, 4)], 0, 2, ops, "cp")
    assert root.issue("cs") == [] and [o[0] for o in ops.log] == ["record", "wait_event", "write"]
    ops.log.clear()
    last = PeerChain(ChainLinks(0, 64, 256, 128, None), [(0, 4)], 1, 2, ops, "cp")
    last.issue("cs")
    last.finish("cs")
    assert [o[0] for o in ops.log] == ["record", "wait_event", "wait", "copy", "write", "record"]
    with pytest.raises(ValueError):
        PeerChain(ChainLinks(0, 64, None, None, None), [(0, 4)], 1, 2, ops, "cp")
    with pytest.raises(ValueError):
        PeerChain(ChainLinks(0, 64, None, None, None), [(0, 4)], 0, 2, ops, "cp")


# ----------------------------------------------------------- multi-process


class _ShmOps:
    """Chain operations on shared memory: addresses are this process's
    virtual addresses of the attached segments."""

    def __init__(self, segments):
        self.regions = [(np.frombuffer(s.buf, dtype=np.uint8).ctypes.data, s.size, s) for s in segments]

    def _view(self, addr, n):
        for base, size, seg in self.regions:
            if base <= addr and addr + n <= base + size:
                return np.frombuffer(seg.buf, dtype=np.uint8)[addr - base: addr - base + n]
        raise AssertionError(f"address {addr:#x}+{n} outside every segment")

    def record(self, stream):
        return None

    def wait_event(self, stream, ev):
        pass

    def wait_geq(self, stream, addr, value):
        flag = self._view(addr, 4).view(np.uint32)
        t0 = time.time()
        while (int(flag[0]) - value) & 0xFFFFFFFF >= 0x80000000:  # cyclic GEQ, as the GPU's
            if time.time() - t0 > 60:
                raise TimeoutError(f"flag {addr:#x} stuck at {int(flag[0])} < {value}")
            time.sleep(1e-4)

    def write(self, stream, addr, value):
        self._view(addr, 4).view(np.uint32)[0] = value

    def copy(self, stream, dst, src, n):
        time.sleep(0.02)  # a slow link: a source overwritten too early shows up as a wrong A
        self._view(dst, n)[:] = self._view(src, n)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, shape, lds, k_chunk, overlap, root, out_q):
    import oracle

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    segs = []
    try:
        m, n, k = shape
        lda, ldb, ldc = lds
        plan = make_shard_plan(m, n, k, world, root=root, k_chunk=k_chunk)
        j0, j1 = plan.local(rank)
        a1, b, c = oracle.make_padded_operands(42, m, n, k, lda, ldb, ldc, canary=-9.0)
        a2 = oracle.make_padded_operands(43, m, n, k, lda, ldb, ldc, canary=-9.0)[0]
        drv = ShardedDgemm(plan, rank, overlap=overlap, stream=lambda: "compute",
                           compute=lambda m_, nl, kc, A_, la, B_, lb, C_, lc: oracle.naive(
                               m_, nl, kc, A_, la, B_, lb, C_, lc))
        spans = drv.chain_spans(lda)
        # this rank's A (root: the source; others: NaN until the chain fills it) and flags
        a_seg = shared_memory.SharedMemory(create=True, size=a1.nbytes)
        f_seg = shared_memory.SharedMemory(create=True, size=8 * len(spans))
        segs += [a_seg, f_seg]
        A = np.frombuffer(a_seg.buf, dtype=np.float64)
        A[:] = a1 if rank == root else np.nan
        np.frombuffer(f_seg.buf, dtype=np.uint32)[:] = 0
        names = [None] * world
        dist.all_gather_object(names, (a_seg.name, f_seg.name))
        q = chain_position(rank, root, world)
        pred = (root + q - 1) % world if q > 0 else None
        succ = (root + q + 1) % world if q < world - 1 else None
        def attach(name):
            seg = shared_memory.SharedMemory(name=name)
            segs.append(seg)
            return seg

        addr = lambda seg: np.frombuffer(seg.buf, dtype=np.uint8).ctypes.data
        pa, pf = (attach(names[pred][0]), attach(names[pred][1])) if pred is not None else (None, None)
        sf = attach(names[succ][1]) if succ is not None else None
        links = ChainLinks(addr(a_seg), addr(f_seg), addr(pa) if pa else None, addr(pf) if pf else None,
                           addr(sf) if sf else None)
        drv.attach_chain(PeerChain(links, spans, q, world, _ShmOps(segs), copy_stream="copy"))
        C_local = c[j0 * ldc:j1 * ldc].copy()
        B_local = b[j0 * ldb:j1 * ldb]
        drv.step(A, lda, B_local, ldb, C_local, ldc)
        ok1 = np.array_equal(oracle.valid_region(A, m, k, lda), oracle.valid_region(a1, m, k, lda))
        if rank == root:  # step 1 finished on every successor's side: the source may change
            A[:] = a2
        drv.step(A, lda, B_local, ldb, C_local, ldc)
        ok2 = np.array_equal(oracle.valid_region(A, m, k, lda), oracle.valid_region(a2, m, k, lda))
        dist.barrier()
        out_q.put((rank, j0, j1, C_local.copy(), ok1, ok2))
    finally:
        dist.barrier()
        for s in segs[:2]:  # views into the segments stay alive until exit: unlink only
            s.unlink()
        dist.destroy_process_group()


@pytest.mark.parametrize("world,root,shape,lds,k_chunk,overlap", [
    (2, 0, (37, 300, 71), (44, 76, 40), 32, True),
    (3, 0, (37, 300, 71), (44, 76, 40), 16, True),
    (3, 2, (16, 400, 50), (16, 50, 16), 16, False),
    (4, 1, (29, 520, 90), (31, 90, 29), 32, True),
])
def test_chain_exchange_two_steps_bitwise_equals_oracle(world, root, shape, lds, k_chunk, overlap):
    """Two steps, the root changing A between them: every rank ends with the
    root's A of each step and C = C0 + A1 B + A2 B,
    bitwise the oracle."""
    import oracle

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, shape, lds, k_chunk, overlap, root, q))
             for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    m, n, k = shape
    lda, ldb, ldc = lds
    a1, b, c = oracle.make_padded_operands(42, m, n, k, lda, ldb, ldc, canary=-9.0)
    a2 = oracle.make_padded_operands(43, m, n, k, lda, ldb, ldc, canary=-9.0)[0]
    want = oracle.naive(m, n, k, a1, lda, b, ldb, c.copy(), ldc)
    want = oracle.naive(m, n, k, a2, lda, b, ldb, want, ldc)
    for rank, j0, j1, cl, ok1, ok2 in sorted(results, key=lambda t: t[0]):
        assert ok1 and ok2, f"rank {rank}: A not delivered (step 1 {ok1}, step 2 {ok2})"
        assert np.array_equal(cl[: (j1 - j0) * ldc], want[j0 * ldc: j1 * ldc]), rank
