"""The NCCL plumbing of the multi-GPU driver on the one GPU of the test box:
a world-size-1 NCCL process group drives multi.ShardedDgemm for rank 0 of a
2-way column split, with the A broadcast going through NCCL (rank 0 is the
root, so no data moves, but the collective is issued on NCCL's stream and
every chunk's GEMM waits on its work handle) -- in both schedules.  The
panel must be bitwise the single-GPU call's columns; the timing all-reduce
bench.py uses (MAX over ranks) is exercised too.  Ranks never wait on one
another's kernels here (world size 1)."""

import os
import socket
import subprocess
import sys
import textwrap

import pytest

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = textwrap.dedent("""
    import sys
    import torch
    import torch.distributed as dist
    sys.path.insert(0, {repo!r})
    from paper_1609_00076_b200 import engine
    from paper_1609_00076_b200.multi import ShardedDgemm, make_shard_plan

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    m, n, k = 1000, 1100, 900
    st = torch.cuda.current_stream().cuda_stream
    bufs = [torch.empty(x, dtype=torch.float64, device=dev) for x in (m * k, k * n, m * n)]
    for t, (buf, r, c) in enumerate(zip(bufs, (m, k, m), (k, n, n))):
        engine.fill_random_device(buf.data_ptr(), r, c, r, 11 + t, 0, st)
    a, b, c0 = bufs
    want = c0.clone()
    engine.dgemm_device(m, n, k, a.data_ptr(), m, b.data_ptr(), k, want.data_ptr(), m, st, force_tiled=True)
    plan = make_shard_plan(m, n, k, 2, root=0, k_chunk=256)
    j0, j1 = plan.local(0)

    def bcast(t, src):
        return dist.broadcast(t, src=src, async_op=True)

    for overlap, reserve in ((False, 0), (True, 0), (True, 16)):
        got = c0.clone()
        ShardedDgemm(plan, 0, broadcast=bcast, overlap=overlap, reserve_sms=reserve).step(
            a, m, b[j0 * k:], k, got[j0 * m:], m)
        torch.cuda.synchronize()
        assert torch.equal(got[j0 * m:j1 * m], want[j0 * m:j1 * m]), (overlap, reserve)
    assert engine.set_max_ctas(0) == 0  # the step restored the cap
    # step_host: the panels and (root) A from pinned host memory, A uploaded
    # chunk by chunk into the chunked broadcast, C's panel back to the host
    nloc = j1 - j0
    hA = a.cpu().pin_memory()
    hB = b[j0 * k:j1 * k].cpu().pin_memory()
    for overlap, reserve in ((False, 0), (True, 0), (True, 16)):
        hC = c0[j0 * m:j1 * m].cpu().pin_memory()
        da = torch.full_like(a, float("nan"))
        db = torch.full((k * nloc,), float("nan"), dtype=torch.float64, device=dev)
        dc = torch.full((m * nloc,), float("nan"), dtype=torch.float64, device=dev)
        drv = ShardedDgemm(plan, 0, broadcast=bcast, overlap=overlap, reserve_sms=reserve)
        for rep in range(2):  # twice: the second step reuses the buffers behind the first
            if rep:
                hC.copy_(c0[j0 * m:j1 * m].cpu())
            out = drv.step_host(hA, da, m, hB, db, k, hC, dc, m)
            assert out is hC
            assert torch.equal(hC, want[j0 * m:j1 * m].cpu()), (overlap, reserve, rep)
    assert engine.set_max_ctas(0) == 0
    t = torch.tensor([3.0, 1.0], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dist.barrier()
    assert float(t[0]) == 3.0
    dist.destroy_process_group()
    print("NCCL-OK", j0, j1, len(plan.chunks))
""")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_nccl_world1_sharded_step_bitwise(tmp_path):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    script = tmp_path / "nccl_step.py"
    script.write_text(SCRIPT.format(repo=REPO))
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()), RANK="0", WORLD_SIZE="1",
               LOCAL_RANK="0")
    r = subprocess.run([sys.executable, str(script)], capture_output=True, text=True, env=env, timeout=300)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert "NCCL-OK" in r.stdout


def test_bench_emulated_world_runs_every_n_gt_1_path(tmp_path):
    """bench.py --emulate-world 4 on the one GPU: rank 0's share of a 4-way
    split through the N > 1 code -- every NCCL exchange schedule timed (the
    chain needs peers and is skipped), the compute-only run, step_host for
    e2e, alt_exchange in the line."""
    import json

    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    for key in ("RANK", "WORLD_SIZE", "LOCAL_RANK"):
        env.pop(key, None)
    r = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--emulate-world", "4", "--workload",
                        "cfg2_8192", "--steps", "2", "--warmup", "3", "--no-cpu-baseline", "--e2e-steps", "1",
                        "--k-chunk", "1024"], capture_output=True, text=True, env=env, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["emulated_world"] == 4 and line["n_gpus"] == 1
    assert line["config"]["n_per_gpu"] == 2048 and line["config"]["k_chunk"] == 1024
    names = {line["config"]["exchange"], *line["alt_exchange"]}
    assert names == {"nccl", "nccl-overlap", "nccl-overlap-reserve8"}
    assert line["value"] > 1000 and line["compute_only_ms_per_step"] > 0
    assert line["e2e"]["api"].startswith("ShardedDgemm.step_host") and line["e2e"]["value"] > 0
    assert line["gpu_launches"] > 0 and line["roofline"]["frac"] > 0.3
