"""Data-parallel partitioning of one conv layer over the GPUs of a box
(SURVEY 8(e)): images are independent, so shard by batch; when the batch is
smaller than the world (batch 1), shard by output channel instead (every rank
reads all of x and 1/G of the filters).  No collective on the data path: the
helpers below are for timing (max over ranks) and for gathering results for
checking, outside the timed region."""
from __future__ import annotations


def split(total: int, world: int, rank: int):
    """Balanced contiguous split: (start, count) of rank's share (count may be 0)."""
    base, rem = divmod(total, world)
    start = rank * base + min(rank, rem)
    return start, base + (1 if rank < rem else 0)


def shard(n: int, c_out: int, world: int, rank: int):
    """-> dict(mode, n0, n, co0, co): this rank's slice of a [n] x [c_out] problem."""
    if n >= world:
        n0, nn = split(n, world, rank)
        return {"mode": "batch", "n0": n0, "n": nn, "co0": 0, "co": c_out}
    co0, cc = split(c_out, world, rank)
    return {"mode": "cout", "n0": 0, "n": n, "co0": co0, "co": cc}


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (the timed region's duration) over all ranks."""
    import torch
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized():
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_nhwc(local, full_shape, sh, world: int, device=None):
    """All-gather per-rank NHWC output shards into the full tensor (checking
    only).  Shards are padded to the largest share so all_gather_into_tensor
    sees equal sizes."""
    import torch
    import torch.distributed as dist
    n, h, w, c = full_shape
    if dist.get_backend() == "gloo":   # the gloo validation mode (and the CPU tests): host tensors
        dev_out = local.device
        out = gather_nhwc(local.cpu(), full_shape, sh, world, device="cpu") if local.is_cuda else None
        if out is not None:
            return out.to(dev_out)
    if sh["mode"] == "batch":
        size = split(n, world, 0)[1]
        buf = torch.zeros((size, h, w, c), dtype=local.dtype, device=device)
        buf[: local.shape[0]] = local
        out = torch.empty((world * size, h, w, c), dtype=local.dtype, device=device)
        dist.all_gather_into_tensor(out, buf)
        parts = [out[r * size: r * size + split(n, world, r)[1]] for r in range(world)]
        return torch.cat(parts, 0)
    size = split(c, world, 0)[1]
    buf = torch.zeros((n, h, w, size), dtype=local.dtype, device=device)
    buf[..., : local.shape[3]] = local
    out = torch.empty((world, n, h, w, size), dtype=local.dtype, device=device)
    dist.all_gather_into_tensor(out, buf.unsqueeze(0).contiguous())
    parts = [out[r, ..., : split(c, world, r)[1]] for r in range(world)]
    return torch.cat(parts, 3)
