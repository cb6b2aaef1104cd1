"""Multi-GPU plumbing of one detection round.

One process per GPU.  The B samples of a round are split into P contiguous ranges (every
sample is solved entirely on one rank), the G mesh nodes into P contiguous ranges.  The only
exchange steps are
  * the transpose [G][B/P] (sample-sharded) -> P slabs [G/P][B_p] (node-sharded), one
    all-to-all (north_star);
  * an all-reduce MAX of the 8-byte kappa_max (threshold basis, Z5);
  * an all-reduce SUM of the int32 votes (union over all nodes, Alg. 1 Step 2e P:318).
All three are pure data movement or order-free (MAX, integer SUM), so the results are
bit-identical for every P.  torch.distributed provides the collectives (NCCL on GPUs; gloo in
the CPU tests of this module's index math).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def partition(n: int, P: int, r: int) -> tuple[int, int]:
    """Contiguous balanced range [lo, hi) of rank r: the first n % P ranks get one extra."""
    q, rem = divmod(n, P)
    lo = r * q + min(r, rem)
    return lo, lo + q + (1 if r < rem else 0)


def bounds(n: int, P: int) -> list[int]:
    """[b_0 = 0, b_1, ..., b_P = n] with rank p owning [b_p, b_{p+1})."""
    return [partition(n, P, p)[0] for p in range(P)] + [n]


class Exchange:
    """The collectives of a round for world size P (P = 1: no-ops)."""

    def __init__(self, group=None):
        self.group = group
        self.P = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if self.P > 1 else 0

    def transpose(self, u_local: torch.Tensor, G: int, B: int) -> tuple[torch.Tensor, list[int]]:
        """[G][nb_rank] (samples of this rank, all nodes) -> slabs [P][G_loc][nb_p] (all samples,
        this rank's nodes).  Returns (slab buffer, slab_b0)."""
        sb = bounds(B, self.P)
        if self.P == 1:
            return u_local, sb
        gb = bounds(G, self.P)
        nb = sb[self.rank + 1] - sb[self.rank]
        g_loc = gb[self.rank + 1] - gb[self.rank]
        send = [(gb[q + 1] - gb[q]) * nb for q in range(self.P)]
        recv = [g_loc * (sb[p + 1] - sb[p]) for p in range(self.P)]
        out = torch.empty(sum(recv), dtype=u_local.dtype, device=u_local.device)
        if u_local.is_cuda and dist.get_backend(self.group) == "gloo":
            # gloo has no CUDA all-to-all: the multi-process GPU tests (several ranks sharing one
            # GPU) stage through host memory; NCCL (the product) exchanges device buffers directly
            host = torch.empty(sum(recv), dtype=u_local.dtype)
            dist.all_to_all_single(host, u_local.reshape(-1).cpu(), recv, send, group=self.group)
            out.copy_(host)
            return out, sb
        dist.all_to_all_single(out, u_local.reshape(-1), recv, send, group=self.group)
        return out, sb

    def max_(self, t: torch.Tensor) -> torch.Tensor:
        if self.P > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
        return t

    def sum_(self, t: torch.Tensor) -> torch.Tensor:
        if self.P > 1:
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
        return t

    def barrier(self):
        if self.P > 1:
            dist.barrier(group=self.group)
