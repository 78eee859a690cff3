"""Session sharding and the post-run result gather, including
a world_size-2 gloo run on CPU."""
import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_2603_13289_b200.sessions import gather_records, shard


@pytest.mark.parametrize("n,world", [(64, 1), (64, 2), (64, 8), (7, 3), (3, 8), (0, 2)])
def test_shard_covers_every_session_once(n, world):
    ids = [i for r in range(world) for i in shard(n, world, r)]
    assert ids == list(range(n))
    sizes = [len(shard(n, world, r)) for r in range(world)]
    assert max(sizes) - min(sizes) <= 1


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    recs = [{"session": s, "first_token": 1000 + s, "segments": 2, "selected_total": s % 5, "reuse": 0.75,
             "ttft_ms": 5.0 + rank} for s in shard(n, world, rank)]
    out = gather_records(recs, n, dist)
    dist.barrier()
    if rank == 0:
        q.put(out)
    dist.destroy_process_group()


@pytest.mark.parametrize("n", [64, 5])
def test_gloo_world2_gather(n):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = q.get(timeout=120)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    assert [r["session"] for r in out] == list(range(n))
    assert all(r["first_token"] == 1000 + r["session"] for r in out)
    assert {r["ttft_ns"] for r in out} == ({5_000_000, 6_000_000} if n > 1 else {5_000_000})


def test_bench_gpus_flag_spawns_ranks():
    """`python bench.py --gpus 2` (no torchrun around it) launches 2 ranks itself
    (bench.spawn_ranks -> torch.distributed.run), shards c4's 64 sessions, and
    rank 0 prints one line with every session gathered. The stub impl runs the
    same launcher / shard / barrier / max-over-ranks / all_gather plumbing as
    the engine arm with a CPU no-op session (gloo)."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "stub", "--gpus", "2",
                          "--config", "c4", "--steps", "2"], capture_output=True, text=True, timeout=240, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    rec = json.loads(lines[0])
    assert rec["n_gpus"] == 2 and rec["sessions_per_rank"] == 32
    assert rec["sessions_gathered"] == 64 and rec["gathered_ids"] == list(range(64)) and rec["first_tokens_ok"]
