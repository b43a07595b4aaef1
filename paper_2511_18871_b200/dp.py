"""Data parallelism over prompt groups.

Unit of work = one prompt group (prompt + its G responses = one packed
sequence; pipeline.cpp:42-45 keeps a micro-batch inside one group).  Each rank
holds replicated tri-model weights, runs pack -> tri-model forward -> GRPO loss
-> backward for the groups assigned to it with no communication, and the only
exchange per optimizer step is an NCCL allreduce (sum) of the fp32 gradient and
of the five loss scalars (Pipeline::MicrobatchStats).  The caller then sets the
update divisor to the GLOBAL batch's N*G samples (GradBuffer.set_micro_step_count,
pipeline.cpp:350; parl.train_iteration(world_samples=...)) before apply_update, so
every rank applies the identical update.

Host-side logic here (no GPU needed, tested with gloo on CPU):
  * group_cost / lpt_assign  : longest-processing-time assignment of ragged
                               groups to ranks by the FLOP model of §8d
  * bootstrap_comm           : NCCL unique id from rank 0 to every rank over
                               torch.distributed (any backend; gloo here)
"""
from __future__ import annotations

import heapq
from typing import Iterable, List, Sequence


def group_cost(prompt_len: int, response_lens: Sequence[int], d: int, L: int, F: int, V: int) -> float:
    """Algorithmic FLOPs of one shared-prompt micro-step (tri-model forward +
    policy backward): GEMMs linear in T, attention in allowed pairs, head in
    scored rows."""
    T = prompt_len + sum(response_lens)
    pairs = prompt_len * (prompt_len + 1) / 2 + sum(r * prompt_len + r * (r + 1) / 2 for r in response_lens)
    rows = 1 + sum(r - 1 for r in response_lens)
    gemm = 2.0 * T * L * (4 * d * d + 2 * d * F)
    attn = 4.0 * pairs * d * L
    head = 2.0 * rows * d * V
    return 3 * (gemm + attn + head) + 2 * gemm + 2.5 * attn + 2 * head


def lpt_assign(costs: Sequence[float], world: int) -> List[List[int]]:
    """Greedy LPT: largest group first onto the least-loaded rank.  Ties break
    on the lower rank and the lower group index, so every rank computes the
    same assignment independently."""
    if world < 1:
        raise ValueError("world must be >= 1")
    order = sorted(range(len(costs)), key=lambda i: (-costs[i], i))
    heap = [(0.0, r) for r in range(world)]
    out: List[List[int]] = [[] for _ in range(world)]
    for i in order:
        load, r = heapq.heappop(heap)
        out[r].append(i)
        heapq.heappush(heap, (load + costs[i], r))
    for r in out:
        r.sort()
    return out


def rank_groups(n_groups: int, costs: Iterable[float] | None, world: int, rank: int) -> List[int]:
    """Groups of `rank`: LPT when costs are given (ragged batches), else round-robin."""
    if costs is None:
        return list(range(rank, n_groups, world))
    return lpt_assign(list(costs), world)[rank]


def bootstrap_comm(ctx, rank: int, world: int, make_id=None):
    """Create the NCCL communicator of `ctx` (paper_2511_18871_b200.parl.Context):
    rank 0 draws the unique id, torch.distributed broadcasts it."""
    import torch.distributed as dist

    if world == 1:
        return None
    uid = (make_id or ctx.comm_unique_id)() if rank == 0 else b""
    obj = [uid]
    dist.broadcast_object_list(obj, src=0)
    if ctx is not None:
        ctx.comm_init(obj[0], rank, world)
    return obj[0]
