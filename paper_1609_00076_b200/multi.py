"""jc-sharded multi-GPU my_dgemm: one process per GPU, torch.distributed for
the plumbing, the A broadcast overlapped with the per-rank GEMM chunk by chunk.

Reference mapping.  The reference parallelises loop 3 (ic) or loop 2 (jr)
over threads with a static, contiguous, balanced split (`split_range`,
pkg/src/gemmforge/parallel.py:39-57) and never splits pc, because pc
iterations accumulate into the same C elements (parallel.py:1-12).  Across
GPUs the natural independent loop is loop 5 (jc, goto.py:212): column j of C
depends only on A and column j of B.  So:

  * rank g owns the contiguous column panel [j0_g, j1_g) of B and C
    (`split_columns`, the split_range rule, rounded to the 128-column CTA
    tile) -- B and C are never communicated;
  * A (m x k) lives on `root` and is broadcast -- whole before the GEMM by
    default, or in k-chunks (`k_chunks`, multiples of 16 = the kernel's K
    slab, so chunked accumulation is bitwise the single call) with chunk i+1
    crossing NVLink while chunk i's GEMM runs (overlap=True, see
    ShardedDgemm);
  * each rank runs C_g += A[:, chunk] * B_g[chunk, :] in ascending chunk
    order (my_dgemm_shard), the reference's pc order, so C is bitwise
    identical for every world size;
  * instead of NCCL, A can travel down a copy-engine chain over NVLink peer
    memory (attach_chain, peer.py): no SM is involved, so the transfer
    overlaps the persistent GEMM without competing for SMs.

The compute and broadcast callables are injectable so the host logic runs
under gloo on CPU in tests (tests/test_multi.py); the product path uses the
C ABI and NCCL.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable

__all__ = ["split_columns", "k_chunks", "ShardPlan", "make_shard_plan", "ShardedDgemm"]

TILE_N = 128
K_ALIGN = 16


def split_columns(n: int, parts: int, align: int = TILE_N) -> tuple[tuple[int, int], ...]:
    """Contiguous, balanced column panels, earlier ranks taking the larger
    share (parallel.py:39-57), in units of `align` columns where n allows."""
    if n < 0:
        raise ValueError(f"count must be non-negative, got {n}")
    if parts < 1:
        raise ValueError(f"workers must be positive, got {parts}")
    units = -(-n // align)
    base, rem = divmod(units, parts)
    out, lo = [], 0
    for w in range(parts):
        hi = min(n, lo + (base + (1 if w < rem else 0)) * align)
        out.append((lo, hi))
        lo = hi
    return tuple(out)


def k_chunks(k: int, chunk: int) -> tuple[tuple[int, int], ...]:
    """Ascending k-ranges of `chunk` (rounded up to a multiple of 16)."""
    if k < 1:
        raise ValueError(f"k must be positive, got {k}")
    chunk = max(K_ALIGN, -(-chunk // K_ALIGN) * K_ALIGN)
    return tuple((p, min(k, p + chunk)) for p in range(0, k, chunk))


@dataclass(frozen=True)
class ShardPlan:
    m: int
    n: int
    k: int
    world: int
    root: int
    columns: tuple[tuple[int, int], ...]
    chunks: tuple[tuple[int, int], ...]

    def local(self, rank: int) -> tuple[int, int]:
        return self.columns[rank]


def make_shard_plan(m: int, n: int, k: int, world: int, root: int = 0,
                    k_chunk: int = 2048) -> ShardPlan:
    if min(m, n, k) < 1:
        raise ValueError(f"matrix dims must be positive, got m={m} n={n} k={k}")
    if not 0 <= root < world:
        raise ValueError(f"root {root} outside 0..{world - 1}")
    chunks = k_chunks(k, k_chunk) if world > 1 else ((0, k),)
    return ShardPlan(m, n, k, world, root, split_columns(n, world), chunks)


def a_span(lda: int, m: int, p0: int, p1: int) -> tuple[int, int]:
    """Flat element range holding columns [p0, p1) of A: never past the last
    valid element (matrix.py:58)."""
    return p0 * lda, (p1 - 1) * lda + m


class ShardedDgemm:
    """Per-rank driver.  `A` is a 1-D buffer of >= (k-1)*lda+m doubles on
    every rank (the source on root, a receive buffer elsewhere); B_local /
    C_local hold this rank's column panel (ldb >= k, ldc >= m).

    compute(m, nloc, kc, A_view, lda, B_view, ldb, C_view, ldc) and
    broadcast(tensor, src) -> handle-with-wait() default to the C ABI on the
    current CUDA stream and torch.distributed.broadcast(async_op=True).
    """

    def __init__(self, plan: ShardPlan, rank: int, group=None,
                 compute: Callable | None = None, broadcast: Callable | None = None,
                 force_tiled: bool | None = None, overlap: bool = False, reserve_sms: int = 0,
                 stream: Callable | None = None):
        self.plan, self.rank, self.group = plan, rank, group
        # exchange of A: NCCL broadcast (default) or, once attach_chain() is
        # called, the copy-engine chain over NVLink peer memory (peer.py)
        self.chain = None
        self._stream = stream or self._current_stream
        # overlap=True with reserve_sms > 0 caps the GEMM's persistent grid at
        # (SM count - reserve_sms) CTAs during the step (my_dgemm_set_max_ctas)
        # so the broadcast's NCCL kernels always find free SMs; C is unchanged.
        self.reserve_sms = reserve_sms
        # overlap=True: chunk c+1's broadcast runs under chunk c's GEMM.  Off by
        # default: NCCL's broadcast kernels run on SMs, and the GEMM is a
        # persistent kernel holding one CTA (224 KB of shared memory) on every
        # SM -- a rank whose GEMM started first keeps its NCCL kernel off the
        # SMs for a whole chunk while the peers' NCCL kernels spin on theirs,
        # delaying their GEMM CTAs.  Without multi-GPU hardware to measure the
        # overlap, the default moves all of A first (one broadcast, every rank
        # waits for it) and then runs the GEMM alone; C is bitwise the same.
        self.overlap = overlap
        # Every rank runs the whole problem's kernel family (a narrow panel
        # must not switch kernels: their summation orders differ), which keeps
        # C identical across world sizes.  Only the tiled family is bitwise
        # k-chunk invariant: the other paths get one k-chunk.
        from . import _capi
        from .engine import path as path_of

        self.path = _capi.PATH_TILED if force_tiled else path_of(plan.m, plan.n)
        if self.path != _capi.PATH_TILED and len(plan.chunks) > 1:
            self.plan = plan = ShardPlan(plan.m, plan.n, plan.k, plan.world, plan.root, plan.columns,
                                         ((0, plan.k),))
        self.force_tiled = self.path == _capi.PATH_TILED
        self._compute = compute or self._device_compute
        self._broadcast = broadcast or self._nccl_broadcast

    # -- defaults (GPU) ---------------------------------------------------
    @staticmethod
    def _current_stream():
        import torch

        return torch.cuda.current_stream()

    def _device_compute(self, m, nloc, kc, A, lda, B, ldb, C, ldc):
        import torch

        from .engine import dgemm_device

        dgemm_device(m, nloc, kc, A.data_ptr(), lda, B.data_ptr(), ldb, C.data_ptr(), ldc,
                     torch.cuda.current_stream().cuda_stream, path=self.path)

    def _nccl_broadcast(self, tensor, src):
        import torch.distributed as dist

        return dist.broadcast(tensor, src=src, group=self.group, async_op=True)

    # -- copy-engine chain ------------------------------------------------
    def chain_spans(self, lda: int) -> tuple[tuple[int, int], ...]:
        """A's element span of every k-chunk of this driver's plan: the
        spans a PeerChain for it must be built with."""
        return tuple(a_span(lda, self.plan.m, p0, p1) for (p0, p1) in self.plan.chunks)

    def attach_chain(self, chain) -> None:
        """Exchange A through `chain` (peer.PeerChain over chain_spans())."""
        self.chain = chain

    def _step_chain(self, A, lda, B_local, ldb, C_local, ldc):
        p = self.plan
        nloc = p.local(self.rank)[1] - p.local(self.rank)[0]
        cs = self._stream()
        events = self.chain.issue(cs)
        if self.overlap:  # chunk c's GEMM as soon as chunk c has landed
            for ci, (p0, p1) in enumerate(p.chunks):
                self.chain.wait_chunk(cs, events, ci)
                if nloc > 0:
                    lo, hi = a_span(lda, p.m, p0, p1)
                    self._compute(p.m, nloc, p1 - p0, A[lo:hi], lda, B_local[p0:], ldb, C_local, ldc)
        else:
            for ci in range(len(p.chunks)):
                self.chain.wait_chunk(cs, events, ci)
            if nloc > 0:
                self._compute(p.m, nloc, p.k, A[:a_span(lda, p.m, 0, p.k)[1]], lda, B_local, ldb, C_local, ldc)
        self.chain.finish(cs)
        return C_local

    # -- one step ---------------------------------------------------------
    def step(self, A, lda: int, B_local, ldb: int, C_local, ldc: int, broadcast_a: bool = True):
        p = self.plan
        j0, j1 = p.local(self.rank)
        nloc = j1 - j0
        if self.chain is not None and p.world > 1 and broadcast_a:
            return self._step_chain(A, lda, B_local, ldb, C_local, ldc)
        if not self.overlap:
            if p.world > 1 and broadcast_a:
                lo, hi = a_span(lda, p.m, 0, p.k)
                self._broadcast(A[lo:hi], p.root).wait()  # every rank, root included
            if nloc > 0:
                self._compute(p.m, nloc, p.k, A[:a_span(lda, p.m, 0, p.k)[1]], lda, B_local, ldb, C_local, ldc)
            return C_local
        if self.reserve_sms > 0:
            import torch

            from .engine import set_max_ctas

            sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
            prev = set_max_ctas(max(1, sms - self.reserve_sms))
            try:
                return self._step_overlapped(A, lda, B_local, ldb, C_local, ldc, broadcast_a)
            finally:
                set_max_ctas(prev)
        return self._step_overlapped(A, lda, B_local, ldb, C_local, ldc, broadcast_a)

    def _step_overlapped(self, A, lda, B_local, ldb, C_local, ldc, broadcast_a):
        p = self.plan
        nloc = p.local(self.rank)[1] - p.local(self.rank)[0]
        works = []
        if p.world > 1 and broadcast_a:
            for (p0, p1) in p.chunks:
                lo, hi = a_span(lda, p.m, p0, p1)
                works.append(self._broadcast(A[lo:hi], p.root))
        for ci, (p0, p1) in enumerate(p.chunks):
            if works and self.rank != p.root:
                works[ci].wait()  # stream-ordered wait on the chunk's arrival
            if nloc > 0:
                lo, hi = a_span(lda, p.m, p0, p1)
                self._compute(p.m, nloc, p1 - p0, A[lo:hi], lda, B_local[p0:], ldb, C_local, ldc)
        if works and self.rank == p.root:
            for w in works:
                w.wait()
        return C_local

    # -- one step from host buffers (the end-to-end measurement) ----------
    def step_host(self, hA, A, lda: int, hB_local, B_local, ldb: int, hC_local, C_local, ldc: int):
        """The same step with the operands in (pinned) host memory: every
        rank uploads its B / C panel, the root uploads A chunk by chunk and
        each chunk's broadcast starts as soon as it has landed, the GEMM
        follows the configured schedule, and the C panel comes back to the
        host.  Host-synchronous.  hA is read on the root only; hB_local /
        hC_local are this rank's panels (ldb / ldc pitched like the device
        panels).  The copy-engine chain exchange uploads all of A first."""
        p = self.plan
        nloc = p.local(self.rank)[1] - p.local(self.rank)[0]
        cuda = A.is_cuda
        root = self.rank == p.root
        spans = [a_span(lda, p.m, p0, p1) for (p0, p1) in p.chunks]
        nb, nc = (nloc - 1) * ldb + p.k if nloc else 0, (nloc - 1) * ldc + p.m if nloc else 0
        if cuda:
            import torch

            cs = self._stream()
            up = self._upload_stream(A.device)
            up.wait_stream(cs)  # the buffers are free once the previous step's work is done
            ctx = torch.cuda.stream(up)
        else:
            import contextlib

            ctx = contextlib.nullcontext()
        works, landed = [], []
        with ctx:
            if nloc:
                B_local[:nb].copy_(hB_local[:nb], non_blocking=True)
                C_local[:nc].copy_(hC_local[:nc], non_blocking=True)
            panels = self._record(up) if cuda else None
            for lo, hi in spans:
                if root:
                    A[lo:hi].copy_(hA[lo:hi], non_blocking=True)
                    landed.append(self._record(up) if cuda else None)
                if p.world > 1 and self.chain is None:
                    works.append(self._broadcast(A[lo:hi], p.root))  # NCCL waits on `up` (the upload)
        if cuda:
            cs.wait_event(panels)
        if self.chain is not None and p.world > 1:
            for ev in landed:
                cs.wait_event(ev)
            self._step_chain(A, lda, B_local, ldb, C_local, ldc)
        else:
            def arrived(ci):
                if root:
                    if cuda:
                        cs.wait_event(landed[ci])
                elif works:
                    works[ci].wait()

            if self.overlap:
                for ci, ((p0, p1), (lo, hi)) in enumerate(zip(p.chunks, spans)):
                    arrived(ci)
                    if nloc > 0:
                        self._compute(p.m, nloc, p1 - p0, A[lo:hi], lda, B_local[p0:], ldb, C_local, ldc)
            else:
                for ci in range(len(spans)):
                    arrived(ci)
                if nloc > 0:
                    self._compute(p.m, nloc, p.k, A[:spans[-1][1]], lda, B_local, ldb, C_local, ldc)
            if root and works:
                for w in works:
                    w.wait()
        if nloc:
            hC_local[:nc].copy_(C_local[:nc], non_blocking=cuda)
        if cuda:
            cs.synchronize()
        return hC_local

    def _upload_stream(self, device):
        import torch

        if getattr(self, "_up", None) is None:
            self._up = torch.cuda.Stream(device=device)
        return self._up

    @staticmethod
    def _record(stream):
        import torch

        ev = torch.cuda.Event()
        ev.record(stream)
        return ev

