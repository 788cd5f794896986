"""GPU side of the copy-engine chain exchange (peer.py, csrc/peer.cu).

One B200 per gpurun call, so the ranks of the chain are emulated inside one
process on one GPU: each emulated rank has its own A buffer, flags, copy
stream and compute stream; "peer" addresses are the other rank's device
addresses (the copy engines move the data; no IPC within one process).  The
operations are queued in a topological host order -- all ranks' chain
traffic first (line order), then the GEMMs, then the end-of-step waits -- so
every stream wait's matching write is already queued when the wait is, and
no emulated rank's stream can block another's even if the driver maps their
streams onto one hardware queue.  No kernel waits on anything.

The IPC export/open path runs across two processes on the GPU with no
device-side wait between them (one process copies from and writes a flag
into the other's memory; a host barrier orders them)."""

import os
import socket

import pytest

from paper_1609_00076_b200 import _capi, engine
from paper_1609_00076_b200.multi import a_span, make_shard_plan
from paper_1609_00076_b200.peer import ChainLinks, CudaChainOps, PeerChain, chain_position

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    _capi.load()
    return torch


@pytest.mark.timeout(300)
@pytest.mark.parametrize("world,root,shape,k_chunk,overlap", [
    (3, 0, (640, 1500, 1000), 256, True),
    (4, 1, (1000, 2000, 700), 128, True),
    (2, 1, (513, 900, 333), 64, False),
    (8, 0, (700, 1111, 900), 256, True),
])
def test_emulated_chain_two_steps_bitwise(torch_cuda, world, root, shape, k_chunk, overlap):
    torch = torch_cuda
    m, n, k = shape
    plan = make_shard_plan(m, n, k, world, root=root, k_chunk=k_chunk)
    spans = [a_span(m, m, p0, p1) for (p0, p1) in plan.chunks]
    seeds = [engine.operand_seed(42, r, m, n, k) for r in (1, 2, 3)]
    st0 = torch.cuda.current_stream().cuda_stream
    a_src = [torch.empty(m * k, dtype=torch.float64, device="cuda") for _ in range(2)]
    for i, t in enumerate(a_src):
        engine.fill_random_device(t.data_ptr(), m, k, m, seeds[0] + i, 0, st0)
    B = torch.empty(k * n, dtype=torch.float64, device="cuda")
    C0 = torch.empty(m * n, dtype=torch.float64, device="cuda")
    engine.fill_random_device(B.data_ptr(), k, n, k, seeds[1], 0, st0)
    engine.fill_random_device(C0.data_ptr(), m, n, m, seeds[2], 0, st0)
    want = C0.clone()
    for t in a_src:  # the single-GPU calls: C0 + A1 B + A2 B
        engine.dgemm_device(m, n, k, t.data_ptr(), m, B.data_ptr(), k, want.data_ptr(), m, st0)
    torch.cuda.synchronize()

    ops = CudaChainOps()
    A = [torch.full((m * k,), float("nan"), dtype=torch.float64, device="cuda") for _ in range(world)]
    A[root].copy_(a_src[0])
    flags = [torch.zeros(2 * len(spans), dtype=torch.int32, device="cuda") for _ in range(world)]
    torch.cuda.synchronize()
    by_pos = sorted(range(world), key=lambda r: chain_position(r, root, world))
    chains, cstreams = {}, {}
    for q, r in enumerate(by_pos):
        pred = by_pos[q - 1] if q > 0 else None
        succ = by_pos[q + 1] if q < world - 1 else None
        links = ChainLinks(A[r].data_ptr(), flags[r].data_ptr(),
                           A[pred].data_ptr() if pred is not None else None,
                           flags[pred].data_ptr() if pred is not None else None,
                           flags[succ].data_ptr() if succ is not None else None)
        chains[r] = PeerChain(links, spans, q, world, ops, torch.cuda.Stream())
        cstreams[r] = torch.cuda.Stream()
    C = C0.clone()
    for step in range(2):
        if step == 1:  # the root's A changes between steps, on its compute stream, no host sync:
            # stream order after the root's finish() (its successor has pulled step 0)
            with torch.cuda.stream(cstreams[root]):
                A[root].copy_(a_src[1])
        events = {r: chains[r].issue(cstreams[r]) for r in by_pos}
        for r in by_pos:
            j0, j1 = plan.local(r)
            cs = cstreams[r]
            chunks = plan.chunks if overlap else ((0, k),)
            for ci, (p0, p1) in enumerate(chunks):
                if overlap:
                    chains[r].wait_chunk(cs, events[r], ci)
                else:
                    for cj in range(len(plan.chunks)):
                        chains[r].wait_chunk(cs, events[r], cj)
                if j1 > j0:
                    lo = p0 * m
                    engine.dgemm_device(m, j1 - j0, p1 - p0, A[r].data_ptr() + 8 * lo, m,
                                        B.data_ptr() + 8 * (j0 * k + p0), k, C.data_ptr() + 8 * j0 * m, m,
                                        cs.cuda_stream)
        for r in by_pos:
            chains[r].finish(cstreams[r])
        torch.cuda.synchronize()
        for r in range(world):
            assert torch.equal(A[r], a_src[step]), (step, r)
    assert torch.equal(C, want)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _ipc_worker(rank, port, q):
    import ctypes

    import torch
    import torch.distributed as dist

    from paper_1609_00076_b200.peer import _export, _IpcMap

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=2)
    try:
        torch.cuda.set_device(0)
        lib = _capi.load()
        n = (1 << 20) + 3
        buf = torch.arange(n, dtype=torch.float64, device="cuda") * (rank + 1)
        flags = torch.zeros(4, dtype=torch.int32, device="cuda")
        view = buf[5:]  # an interior pointer: export = allocation handle + offset
        torch.cuda.synchronize()
        table = [None, None]
        dist.all_gather_object(table, (_export(view.data_ptr()), _export(flags.data_ptr())))
        ok = True
        if rank == 1:
            ipc = _IpcMap()
            peer_view = ipc.resolve(*table[0][0])
            peer_flags = ipc.resolve(*table[0][1])
            dst = torch.empty(n - 5, dtype=torch.float64, device="cuda")
            st = torch.cuda.current_stream().cuda_stream
            _capi.check(lib.my_dgemm_copy_async(dst.data_ptr(), peer_view, 8 * (n - 5), st))
            _capi.check(lib.my_dgemm_signal_write(st, peer_flags + 8, 77))
            torch.cuda.synchronize()
            ok = torch.equal(dst, torch.arange(5, n, dtype=torch.float64, device="cuda"))
            ipc.close()
        dist.barrier()  # rank 1's copy and flag write are complete
        if rank == 0:
            ok = flags.cpu().tolist() == [0, 0, 77, 0]
        st = ctypes.c_void_p(0)
        bad = lib.my_dgemm_signal_write(st, flags.data_ptr() + 2, 1)  # misaligned flag address
        ok = ok and bad == -2
        # connect_chain: the collective set-up bench.py --exchange chain uses (no step is run)
        from paper_1609_00076_b200.peer import connect_chain

        chain, close = connect_chain(buf, [(0, 100), (100, 200)], rank, 2, root=0)
        L = chain.links
        if rank == 0:
            ok = ok and chain.position == 0 and L.a_pred is None and L.flags_succ is not None
        else:
            ok = ok and chain.position == 1 and L.flags_succ is None
            got = torch.empty(200, dtype=torch.float64, device="cuda")
            _capi.check(lib.my_dgemm_copy_async(got.data_ptr(), L.a_pred, 1600, 0))
            torch.cuda.synchronize()
            ok = ok and torch.equal(got, torch.arange(200, dtype=torch.float64, device="cuda"))
        close()
        q.put((rank, bool(ok)))
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_ipc_export_open_copy_and_remote_flag_write(torch_cuda):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ipc_worker, args=(r, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res == {0: True, 1: True}
