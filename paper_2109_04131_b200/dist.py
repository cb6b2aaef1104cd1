"""Multi-GPU plumbing of one detection round.

One process per GPU.  The B samples of a round are split into P contiguous ranges (every
sample is solved entirely on one rank), the G mesh nodes into P contiguous ranges.  The only
exchange steps are
  * the transpose [G][B/P] (sample-sharded) -> P slabs [G/P][B_p] (node-sharded), one
    all-to-all (north_star);
  * an all-reduce MAX of the 8-byte kappa_max (threshold basis, Z5);
  * an all-reduce SUM of the int32 votes (union over all nodes, Alg. 1 Step 2e P:318).
All three are pure data movement or order-free (MAX, integer SUM), so the results are
bit-identical for every P.

The product runs them inside libusfft (usfft_transpose, usfft_detect_select,
usfft_detect_union over the library's own NCCL communicator): this module only bootstraps the
communicator id over torch.distributed (bootstrap_id).  TorchExchange performs the same three
steps with torch.distributed for process groups the library cannot use (gloo: ranks sharing one
GPU in the multi-process tests, CPU-only index-math tests).
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


def bootstrap_id(group=None) -> bytes:
    """The 128-byte ncclUniqueId of the library's communicator: made on rank 0 by libusfft and
    broadcast over the (initialised) torch.distributed process group."""
    from . import binding
    rank = dist.get_rank(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" else "cpu"
    buf = torch.zeros(128, dtype=torch.uint8, device=dev)
    if rank == 0:
        buf.copy_(torch.frombuffer(bytearray(binding.usfft_comm_unique_id()), dtype=torch.uint8))
    dist.broadcast(buf, src=0, group=group)
    return bytes(buf.cpu().numpy().tobytes())


class TorchExchange:
    """The collectives of a round through torch.distributed, for world size P (P = 1: no-ops).
    Only for process groups the library's communicator cannot serve (gloo)."""

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
