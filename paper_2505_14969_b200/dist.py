"""Multi-GPU plumbing for the tree-verify path.

The path partitions with no exchange step inside it: trees are independent
problems and SSM heads are independent given B, C and the tree (accept uses
replicated verifier tokens; commit is per head).  Two layouts:

* batch sharding (default): rank r verifies its own trees -> no data-path
  collective, weak scaling;
* head sharding: rank r owns heads [h_lo, h_hi) of every tree (whole groups
  when G > 1); a layer that needs the full y all-gathers the per-rank head
  shards over NCCL (`gather_heads`).  Commit stays local (the state of a head
  lives on the rank that owns the head).

Only torch.distributed calls live here; no arithmetic of the method.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous near-equal split of n items: [lo, hi) for `rank`."""
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def shard_heads(n_heads: int, n_groups: int, world: int, rank: int) -> tuple[int, int]:
    """Heads [lo, hi) of `rank`.  With G > 1 groups and world <= G, whole groups are
    assigned so that B/C stay group-local; otherwise heads are split evenly and
    must not straddle a group boundary (checked)."""
    hpg = n_heads // n_groups
    if n_groups > 1 and world <= n_groups:
        g_lo, g_hi = shard_range(n_groups, world, rank)
        return g_lo * hpg, g_hi * hpg
    lo, hi = shard_range(n_heads, world, rank)
    if hi > lo and lo // hpg != (hi - 1) // hpg:
        raise ValueError("head shard straddles a group boundary; choose world | (H/G)")
    return lo, hi


def gather_heads(y_local: torch.Tensor, group=None) -> torch.Tensor:
    """All-gather head shards y_local [B][T][H_r][P] (equal H_r on every rank) into
    [world][B][T][H_r][P]; rank-major = head-major for contiguous shards."""
    world = dist.get_world_size(group)
    shp = tuple(y_local.shape)
    out = torch.empty((world * shp[0],) + shp[1:], dtype=y_local.dtype, device=y_local.device)
    dist.all_gather_into_tensor(out, y_local.contiguous(), group=group)
    return out.view((world,) + shp)


def max_over_ranks(value: float, device) -> float:
    """Max of a scalar over all ranks (timing: the slowest rank defines the step)."""
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
