"""Multi-GPU batch plumbing (A10 / §8(e)): instances are partitioned over ranks
(one process per GPU) and each rank's results travel as fixed 64-B records
gathered with ONE collective (NCCL all_gather on GPUs, gloo in the CPU tests).
No collective touches the data path: every rank solves its own instances."""
from __future__ import annotations

import numpy as np

RECORD_FIELDS = ("instance", "status", "flow", "cut_capacity", "rounds", "global_relabels", "pushes", "relabels")


def partition(total: int, world: int, rank: int):
    """Contiguous block [lo, hi) of instance ids owned by `rank` (sizes differ by <= 1)."""
    base, extra = divmod(total, world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return lo, hi


def partition_weighted(weights, world: int, rank: int):
    """Contiguous block [lo, hi) of instance ids for `rank`, balanced by weight (the edge
    count m of every instance): boundary r sits where the running weight is
    closest to r/world of the total, every rank keeping at least one instance when there
    are enough of them."""
    w = np.asarray(weights, np.float64)
    total = w.shape[0]
    if world <= 1 or total == 0:
        return (0, total) if rank == 0 else (total, total)
    cum = np.concatenate([[0.0], np.cumsum(w)])
    cuts = [0]
    for r in range(1, world):
        target = cum[-1] * r / world
        i = int(np.argmin(np.abs(cum - target)))
        lo_ok = cuts[-1] + (1 if total >= world else 0)       # at least one per rank
        hi_ok = total - (world - r if total >= world else 0)  # leave one for each later rank
        cuts.append(int(min(max(i, lo_ok), hi_ok)))
    cuts.append(total)
    return cuts[rank], cuts[rank + 1]


def make_records(ids, flows, cuts, stats=None, status=0) -> np.ndarray:
    """int64[k, 8] records (64 B each)."""
    k = len(ids)
    r = np.zeros((k, len(RECORD_FIELDS)), np.int64)
    r[:, 0] = ids
    r[:, 1] = status
    r[:, 2] = flows
    r[:, 3] = cuts
    if stats:
        r[:, 4] = stats.get("rounds", 0)
        r[:, 5] = stats.get("global_relabels", 0)
        r[:, 6] = stats.get("pushes", 0)
        r[:, 7] = stats.get("relabels", 0)
    return r


def gather_records(local, total: int, world: int, device=None):
    """All-gather every rank's records; returns int64[total, 8] ordered by instance id.
    `local` is a torch int64 tensor [k_local, 8] on the collective's device.  When a
    process group is initialised the collective runs at every world size (world 1 too)."""
    import torch
    import torch.distributed as dist
    if world == 1 and not (dist.is_available() and dist.is_initialized()):
        out = local
    else:
        cap = -(-total // world) if world > 0 else total
        cap = max(cap, int(local.shape[0]))
        # ranks may own different counts (weighted partition): pad to the largest
        if world > 1:
            n_local = torch.tensor([local.shape[0]], dtype=torch.int64, device=local.device)
            sizes = [torch.empty_like(n_local) for _ in range(world)]
            dist.all_gather(sizes, n_local)
            cap = max(int(s.item()) for s in sizes)
        buf = torch.full((cap, local.shape[1]), -1, dtype=torch.int64, device=local.device)
        buf[:local.shape[0]] = local
        parts = [torch.empty_like(buf) for _ in range(world)]
        dist.all_gather(parts, buf)
        out = torch.cat(parts)
        out = out[out[:, 0] >= 0]
    out = out[torch.argsort(out[:, 0])]
    assert out.shape[0] == total and bool((out[:, 0] == torch.arange(total, device=out.device)).all())
    return out


def gather_records_async(local, counts, world: int, out=None):
    """The timed-loop form of gather_records: every rank knows all ranks' record counts
    (`counts`, from the deterministic partition), so the records are padded to max(counts)
    and gathered with ONE all_gather_into_tensor, with no host synchronisation (no size
    exchange, no masking or sorting on the host).  Returns the padded int64[world * cap, 8]
    tensor; order_records() strips and orders it after the timed region."""
    import torch
    import torch.distributed as dist
    cap = max(int(c) for c in counts)
    k = int(local.shape[0])
    if k < cap:
        local = torch.cat([local, torch.full((cap - k, local.shape[1]), -1, dtype=local.dtype, device=local.device)])
    if world == 1 and not (dist.is_available() and dist.is_initialized()):
        return local
    if out is None:
        out = torch.empty((world * cap, local.shape[1]), dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(out, local)
    return out


def order_records(gathered, total: int):
    """Strip the padding of gather_records_async's result and order by instance id (checked)."""
    import torch
    out = gathered[gathered[:, 0] >= 0]
    out = out[torch.argsort(out[:, 0])]
    assert out.shape[0] == total and bool((out[:, 0] == torch.arange(total, device=out.device)).all())
    return out
