"""Session sharding across GPUs and the post-run result gather.

The reference runs independent workflow instances that "may run in parallel"
 and share nothing; sessions are the unit of
parallelism, contiguous blocks of sessions per GPU, one process per GPU, no
collective on the hot path. After the timed region, fixed-size per-session
records (first token id, reuse rates, selection counts, TTFT) are gathered to
rank 0 with one all_gather over NCCL (NVLink) -- gloo in the CPU tests.
"""
import numpy as np

RECORD_FIELDS = ("session", "first_token", "segments", "selected_total", "reuse_x1e6", "ttft_ns")


def shard(n_sessions, world, rank):
    """Contiguous block of session ids owned by `rank` (sizes differ by <= 1)."""
    if n_sessions < 0 or world < 1 or not 0 <= rank < world:
        raise ValueError("bad shard request")
    base, extra = divmod(n_sessions, world)
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


def pack_records(records):
    """List of dicts -> int64 [n, len(RECORD_FIELDS)]."""
    out = np.zeros((len(records), len(RECORD_FIELDS)), np.int64)
    for i, r in enumerate(records):
        out[i] = [int(r["session"]), int(r["first_token"]), int(r.get("segments", 0)),
                  int(r.get("selected_total", 0)), int(round(r.get("reuse", 0.0) * 1e6)),
                  int(round(r.get("ttft_ms", 0.0) * 1e6))]
    return out


def gather_records(records, n_sessions, dist=None, device="cpu"):
    """All-gather every rank's packed records; returns all sessions' records
    sorted by session id (on every rank). `dist` is torch.distributed or None."""
    local = pack_records(records)
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        table = local
    else:
        import torch
        world = dist.get_world_size()
        width = -(-n_sessions // world)  # max shard size
        buf = np.full((width, len(RECORD_FIELDS)), -1, np.int64)
        buf[: len(local)] = local
        t = torch.from_numpy(buf).to(device)
        parts = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(parts, t)
        table = np.concatenate([p.cpu().numpy() for p in parts])
        table = table[table[:, 0] >= 0]
    table = table[np.argsort(table[:, 0], kind="stable")]
    return [dict(zip(RECORD_FIELDS, map(int, row))) for row in table]
