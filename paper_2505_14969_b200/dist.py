"""Multi-GPU plumbing for the tree-verify path.

The path partitions with no exchange step inside it: trees are independent
problems and SSM heads are independent given B, C and the tree (accept uses
replicated verifier tokens; commit is per head).  Two layouts:

* batch sharding (default): rank r verifies its own trees -> no data-path
  collective, weak scaling;
* head sharding: rank r owns heads [h_lo, h_hi) of every tree (whole groups
  when G > 1); the layer's consumer needs the full y on every rank.
  `FullY` provides it: with peer-mapped symmetric memory (torch symmetric
  memory over NVLink / NVSwitch) the scan epilogue itself stores each y tile
  into every rank's full-y buffer (stree_replay_scan_sharded, include/stree.h)
  and one device-side barrier publishes the stores; without it, the scan
  writes a local shard and `gather_heads` all-gathers over NCCL.  Commit stays
  local (the state of a head lives on the rank that owns the head).

Only torch.distributed plumbing lives here; no arithmetic of the method.
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


def heads_to_layer(g: torch.Tensor) -> torch.Tensor:
    """[world][B][T][H_r][P] (gather_heads) -> the layer's [B][T][world·H_r][P] (contiguous shards)."""
    w, B, T, Hr, P = g.shape
    return g.permute(1, 2, 0, 3, 4).reshape(B, T, w * Hr, P)


class FullY:
    """Full-y buffers [L][B][T][H][P] of L head-sharded layers on every rank.

    mode "p2p": one symmetric-memory allocation (torch.distributed._symmetric_memory) rendezvoused over the
    group; `peers(l)` are the device addresses of layer l's buffer on every rank (peer-mapped), the scan
    epilogue writes into all of them, `publish()` is the device-side barrier that makes the stores visible.
    mode "nccl": a plain local buffer per layer; the caller scans into a local shard and calls `gather()`.
    """

    def __init__(self, L, B, T, H, P, dtype, device, group=None, prefer_p2p=True, force_p2p=False):
        self.L, self.shape = L, (B, T, H, P)
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.mode, self.handle = "nccl", None
        self.error = None
        if prefer_p2p and (self.world > 1 or force_p2p):   # force_p2p: exercise the path on one rank
            try:
                import torch.distributed._symmetric_memory as symm_mem
                buf = symm_mem.empty((L, B, T, H, P), dtype=dtype, device=device)
                grp = group if group is not None else dist.group.WORLD
                self.handle = symm_mem.rendezvous(buf, grp)
                self.buf = buf
                self.mode = "p2p"
            except Exception as exc:   # no symmetric memory on this build / topology: NCCL all-gather
                self.error = f"{type(exc).__name__}: {exc}"
                self.handle = None
        if self.mode != "p2p":
            self.buf = torch.empty((L, B, T, H, P), dtype=dtype, device=device)
        self.layer_bytes = self.buf[0].numel() * self.buf.element_size()

    def peers(self, layer: int) -> list[int]:
        """Device addresses of layer `layer`'s full y on every rank (rank order); this rank's own in "nccl"."""
        if self.mode == "p2p":
            return [int(p) + layer * self.layer_bytes for p in self.handle.buffer_ptrs]
        return [self.buf[layer].data_ptr()]

    def publish(self):
        """p2p: device-side barrier over the group on the current stream (every rank's epilogue stores done and
        visible before anything after it reads the full y)."""
        if self.mode == "p2p":
            self.handle.barrier(channel=0)

    def gather(self, layer: int, y_local: torch.Tensor):
        """nccl: all-gather of this rank's shard [B][T][H_r][P] into the layer's full y."""
        g = gather_heads(y_local, self.group)
        self.buf[layer].copy_(heads_to_layer(g))
