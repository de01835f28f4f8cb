"""Snapshot sharding across GPUs: one process per GPU, no per-iteration communication.

Snapshots are independent (same geometry, Lambda and mu; per-snapshot tau), so
rank r solves the contiguous slice [r*B/P, (r+1)*B/P) and the only collective is
one gather to rank 0 after the loop: recovered spectra and peak
lists, over NCCL (NVLink/NVSwitch) on GPUs or gloo in the CPU tests.
"""

import os

import torch
import torch.distributed as dist


def shard_bounds(total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [lo, hi) slice of `total` items for `rank` of `world` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank / world size")
    base, rem = divmod(total, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def env_rank_world() -> tuple[int, int, int]:
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


def init(backend: str | None = None) -> tuple[int, int, int]:
    """Initialise torch.distributed from the torchrun environment (no-op for world 1)."""
    rank, world, local = env_rank_world()
    if world > 1 and not dist.is_initialized():
        if backend is None:
            backend = "nccl" if torch.cuda.is_available() else "gloo"
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if backend == "nccl":
            torch.cuda.set_device(local)
            dist.init_process_group(backend, device_id=torch.device(f"cuda:{local}"))
        else:
            dist.init_process_group(backend)
    elif torch.cuda.is_available():
        torch.cuda.set_device(local)
    return rank, world, local


def gather_rows(local: torch.Tensor, total_rows: int, root: int = 0):
    """Gather row-sharded tensors (dim 0 split by shard_bounds) to `root`.

    Returns the (total_rows, ...) tensor on root and None elsewhere.  Uneven shards
    are padded to the largest shard for the single all-gather-into-tensor call.
    """
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return local
    world, rank = dist.get_world_size(), dist.get_rank()
    biggest = max(shard_bounds(total_rows, r, world)[1] - shard_bounds(total_rows, r, world)[0]
                  for r in range(world))
    pad = torch.zeros((biggest,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    if local.is_complex():
        pad = torch.view_as_real(pad)
    flat = torch.empty((world * pad.shape[0],) + tuple(pad.shape[1:]), dtype=pad.dtype, device=pad.device)
    dist.all_gather_into_tensor(flat, pad)
    out = flat.view((world,) + tuple(pad.shape))
    if rank != root:
        return None
    parts = []
    for r in range(world):
        lo, hi = shard_bounds(total_rows, r, world)
        parts.append(out[r, : hi - lo])
    full = torch.cat(parts, dim=0)
    return torch.view_as_complex(full.contiguous()) if local.is_complex() else full


def max_over_ranks(value: float) -> float:
    """Max of a host scalar over ranks (multi-GPU timings are reported as the max)."""
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return value
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" else torch.device("cpu")
    t = torch.tensor([value], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
