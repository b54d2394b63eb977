"""Expert-sharded serving across the GPUs of one box.

Experts are the independent units: the base model is replicated on every GPU and
expert e lives on rank `e mod G` (`Placement`).  A request is routed (router.classify,
or given) to exactly one expert and decode tokens never mix experts (PAPER.md:136-137,
SPEC.md:546), so the data path has NO collective: rank 0 enqueues each request to its
owner's queue (`dispatch`, a host-side control message over the process group), every
rank runs its own fused multi-expert batches on its own GPU, and results return over
host memory (`collect`).  torch.distributed carries only these small host objects
(gloo or nccl); the per-token tensors never cross GPUs.
"""

from __future__ import annotations

from dataclasses import dataclass

__all__ = ["Placement", "partition", "dispatch", "collect", "ShardedService"]


@dataclass(frozen=True)
class Placement:
    """Expert -> owner rank; `mod` = e mod G."""
    n_experts: int
    world_size: int

    def __post_init__(self):
        if self.n_experts < 1 or self.world_size < 1:
            raise ValueError("need >= 1 expert and >= 1 rank")

    def owner(self, expert: int) -> int:
        if not 0 <= expert < self.n_experts:
            raise ValueError(f"expert id {expert} out of range")
        return expert % self.world_size

    def local_experts(self, rank: int) -> list:
        return [e for e in range(self.n_experts) if e % self.world_size == rank]

    def local_index(self, expert: int) -> int:
        """Slot of `expert` in its owner's local expert list."""
        return expert // self.world_size


def partition(requests, placement: Placement) -> list:
    """requests: iterable of (request_id, expert_id, payload) -> per-rank lists, request
    order preserved within each rank."""
    out = [[] for _ in range(placement.world_size)]
    for req in requests:
        out[placement.owner(int(req[1]))].append(req)
    return out


def dispatch(requests, placement: Placement, rank: int, group=None, src: int = 0) -> list:
    """Rank `src` partitions its request list by owner and hands each rank its share
    (host control message).  Returns this rank's requests."""
    import torch.distributed as dist
    ws = placement.world_size
    if ws == 1:
        return list(requests) if rank == src else []
    scatter = partition(requests, placement) if rank == src else None
    out = [None]
    dist.scatter_object_list(out, scatter, src=src, group=group)
    return out[0]


def collect(local_results: dict, placement: Placement, rank: int, group=None, dst: int = 0):
    """Gather {request_id: result} from every rank onto `dst` (host memory)."""
    import torch.distributed as dist
    if placement.world_size == 1:
        return dict(local_results)
    gathered = [None] * placement.world_size if rank == dst else None
    dist.gather_object(dict(local_results), gathered, dst=dst, group=group)
    if rank != dst:
        return None
    merged = {}
    for part in gathered:
        for k, v in part.items():
            if k in merged:
                raise RuntimeError(f"request {k} served twice")
            merged[k] = v
    return merged


class ShardedService:
    """One rank's share of the box: `serve(local_requests) -> {request_id: result}` runs
    this rank's experts only (e.g. MistralMultiExpert.decode over the local batch)."""

    def __init__(self, placement: Placement, rank: int, serve, group=None):
        self.placement, self.rank, self.serve, self.group = placement, rank, serve, group

    def step(self, requests=None, src: int = 0):
        local = dispatch(requests or [], self.placement, self.rank, self.group, src)
        for req in local:
            if self.placement.owner(int(req[1])) != self.rank:
                raise RuntimeError("request dispatched to a rank that does not own its expert")
        results = self.serve(local) if local else {}
        return collect(results, self.placement, self.rank, self.group, src)
