"""Copy-engine chain broadcast of A over NVLink peer memory.

The jc-sharded driver (multi.py) has one exchange step: A (m x k,
on the root rank) must reach every rank.  The reference has no counterpart --
its threads share A in one address space (pkg/src/gemmforge/parallel.py:
108-243).  NCCL's broadcast runs as kernels on SMs, which the persistent GEMM
(one 224 KB-shared-memory CTA on every SM) keeps busy, so an NCCL broadcast
overlapped with the GEMM fights it for SMs.  The chain
moves A with the DMA copy engines instead, which need no SM:

  * the ranks form a line from the root: position q = (rank - root) mod world;
  * per k-chunk c (the plan's chunks, ascending), the rank at position q >= 1
    waits until its own flag ready[c] reaches the step number, pulls chunk c
    from position q - 1's A over NVLink (cudaMemcpyAsync on an IPC-mapped
    peer pointer), then writes freed[c] = step into q - 1's flags ("done
    reading your chunk") and, if it has a successor, ready[c] = step into
    q + 1's flags; the root only writes its successor's ready flags;
  * the GEMM of chunk c waits (event) for that chunk's copy, so chunk c + 1
    crosses NVLink while chunk c is multiplied;
  * at the end of a step the rank's compute stream waits until its successor
    has pulled every chunk (its own freed flags), so once a step completes in
    stream order, the rank's A may be overwritten again (next step, or by the
    caller).

Waits and writes are stream memory operations on 32-bit device flags (the
GPU front end executes them; no kernel spins).  A rank only WAITS on its own
flags and only WRITES its neighbours'.  Flag values are the step number, so
they never need resetting; waits compare cyclically (GEQ).

Deadlock freedom: every wait is on a write that the predecessor (ready) or
the successor (freed) issues after waits that depend only on ranks earlier in
the line for the same step, or on earlier steps.

`PeerChain` holds the protocol only; the operations come from an `ops`
object (`CudaChainOps` on the GPU, a shared-memory fake in
tests/test_peer_chain.py, which runs it across real processes on the CPU).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Any, Sequence

__all__ = ["ChainLinks", "PeerChain", "CudaChainOps", "chain_position", "connect_chain"]

FLAG_BYTES = 4


def chain_position(rank: int, root: int, world: int) -> int:
    """Position of `rank` on the line that starts at `root`."""
    if not 0 <= root < world or not 0 <= rank < world:
        raise ValueError(f"rank {rank} / root {root} outside 0..{world - 1}")
    return (rank - root) % world


@dataclass(frozen=True)
class ChainLinks:
    """Addresses one rank needs (plain integers: device addresses on the GPU).

    a_local      this rank's A buffer (element 0)
    flags_local  this rank's flags: ready[0..C) then freed[0..C), uint32
    a_pred       the predecessor's A buffer (None at the root)
    flags_pred   the predecessor's flags (None at the root)
    flags_succ   the successor's flags (None at the end of the line)
    """

    a_local: int
    flags_local: int
    a_pred: int | None
    flags_pred: int | None
    flags_succ: int | None


class PeerChain:
    """One rank's side of the chain for a fixed list of A element spans
    (`spans[c] = (lo, hi)` element offsets of chunk c, 8-byte elements)."""

    def __init__(self, links: ChainLinks, spans: Sequence[tuple[int, int]], position: int, world: int, ops: Any,
                 copy_stream: Any):
        if not 0 <= position < world:
            raise ValueError(f"position {position} outside 0..{world - 1}")
        if (position > 0) != (links.a_pred is not None and links.flags_pred is not None):
            raise ValueError("a predecessor's A and flags are needed exactly when position > 0")
        if (position < world - 1) != (links.flags_succ is not None):
            raise ValueError("a successor's flags are needed exactly when position < world - 1")
        self.links, self.spans, self.position, self.world = links, tuple(spans), position, world
        self.ops, self.copy_stream = ops, copy_stream
        self.step = 0  # the step number of the last issue(); flags start at 0
        nc = len(self.spans)
        self._ready = lambda base, c: base + FLAG_BYTES * c
        self._freed = lambda base, c: base + FLAG_BYTES * (nc + c)

    @property
    def has_pred(self) -> bool:
        return self.position > 0

    @property
    def has_succ(self) -> bool:
        return self.position < self.world - 1

    def issue(self, compute_stream) -> list:
        """Queue this step's chain traffic; returns one event per chunk that
        the compute stream must wait on before using that chunk of A (empty
        at the root, whose A is the source)."""
        ops, cs, L = self.ops, self.copy_stream, self.links
        self.step = s = (self.step + 1) & 0xFFFFFFFF
        # everything queued on the compute stream so far (A written, the
        # previous step's end) happens before this step's traffic
        ops.wait_event(cs, ops.record(compute_stream))
        events = []
        for c, (lo, hi) in enumerate(self.spans):
            if self.has_pred:
                ops.wait_geq(cs, self._ready(L.flags_local, c), s)
                ops.copy(cs, L.a_local + 8 * lo, L.a_pred + 8 * lo, 8 * (hi - lo))
                ops.write(cs, self._freed(L.flags_pred, c), s)
                events.append(ops.record(cs))
            if self.has_succ:
                ops.write(cs, self._ready(L.flags_succ, c), s)
        return events

    def wait_chunk(self, compute_stream, events: list, c: int) -> None:
        if events:
            self.ops.wait_event(compute_stream, events[c])

    def finish(self, compute_stream) -> None:
        """The compute stream waits until the successor has pulled every
        chunk of this step (A may be overwritten after that)."""
        if self.has_succ:
            for c in range(len(self.spans)):
                self.ops.wait_geq(compute_stream, self._freed(self.links.flags_local, c), self.step)


class CudaChainOps:
    """Chain operations on CUDA streams through the C ABI (peer.cu)."""

    def __init__(self):
        import torch

        from . import _capi

        self.torch, self.lib, self.check = torch, _capi.load(), _capi.check

    def record(self, stream):
        ev = self.torch.cuda.Event()
        ev.record(stream)
        return ev

    def wait_event(self, stream, ev) -> None:
        stream.wait_event(ev)

    def wait_geq(self, stream, addr: int, value: int) -> None:
        self.check(self.lib.my_dgemm_signal_wait_geq(stream.cuda_stream, addr, value))

    def write(self, stream, addr: int, value: int) -> None:
        self.check(self.lib.my_dgemm_signal_write(stream.cuda_stream, addr, value))

    def copy(self, stream, dst: int, src: int, nbytes: int) -> None:
        self.check(self.lib.my_dgemm_copy_async(dst, src, nbytes, stream.cuda_stream))


class _IpcMap:
    """Opened IPC allocations of this process, one mapping per allocation
    (two exported buffers may share one cudaMalloc block)."""

    def __init__(self):
        from . import _capi

        self.lib, self.check = _capi.load(), _capi.check
        self.open: dict[bytes, int] = {}

    def resolve(self, handle: bytes, offset: int) -> int:
        import ctypes

        if handle not in self.open:
            p = ctypes.c_void_p()
            self.check(self.lib.my_dgemm_ipc_open(handle, 0, ctypes.byref(p)))
            self.open[handle] = int(p.value)
        return self.open[handle] + offset

    def close(self) -> None:
        for base in self.open.values():
            self.lib.my_dgemm_ipc_close(base, 0)
        self.open.clear()


def _export(ptr: int) -> tuple[bytes, int]:
    import ctypes

    from . import _capi

    lib = _capi.load()
    h = ctypes.create_string_buffer(_capi.IPC_HANDLE_BYTES)
    off = ctypes.c_uint64()
    _capi.check(lib.my_dgemm_ipc_export(ptr, h, ctypes.byref(off)))
    return h.raw, int(off.value)


def connect_chain(A, spans: Sequence[tuple[int, int]], rank: int, world: int, root: int = 0, group=None):
    """Collective (every rank of `group`): allocate this rank's flags, export
    A and the flags by CUDA IPC, exchange the handles over torch.distributed
    and map the neighbours' buffers.  Returns (PeerChain, close)."""
    import torch
    import torch.distributed as dist

    flags = torch.zeros(2 * len(spans), dtype=torch.int32, device=A.device)
    torch.cuda.synchronize(A.device)
    mine = (_export(A.data_ptr()), _export(flags.data_ptr()))
    table: list = [None] * world
    dist.all_gather_object(table, mine, group=group)
    q = chain_position(rank, root, world)
    pred = (root + q - 1) % world if q > 0 else None
    succ = (root + q + 1) % world if q < world - 1 else None
    ipc = _IpcMap()
    links = ChainLinks(
        a_local=A.data_ptr(), flags_local=flags.data_ptr(),
        a_pred=ipc.resolve(*table[pred][0]) if pred is not None else None,
        flags_pred=ipc.resolve(*table[pred][1]) if pred is not None else None,
        flags_succ=ipc.resolve(*table[succ][1]) if succ is not None else None)
    chain = PeerChain(links, spans, q, world, CudaChainOps(), torch.cuda.Stream(A.device))
    chain._keep = flags  # the flags live as long as the chain

    def close():
        torch.cuda.synchronize(A.device)
        dist.barrier(group=group)  # no rank still reads a neighbour's buffers
        ipc.close()

    return chain, close
