"""Multi-GPU stream sharding.

Capture streams are independent TrackState recursions, so a job of
`n_streams` streams is partitioned across ranks (one process per GPU) with
no collective on the data path; every rank batches its streams into every
kernel launch.  Results are gathered to rank 0 at the end of a sequence (or
every K frames) with one collective -- NCCL over NVLink / NVSwitch on GPUs,
gloo on CPU -- the only communication of the tracking job.
"""

from __future__ import annotations

import numpy as np


def assign_streams(n_streams: int, world: int, rank: int, policy: str = "block") -> list:
    """Global stream ids owned by `rank`.  'block': contiguous ranges (the
    bench's seeds rank*S ..); 'round_robin': stream s -> rank s % world."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank / world size")
    if policy == "round_robin":
        return list(range(rank, n_streams, world))
    if policy == "block":
        per, extra = divmod(n_streams, world)
        start = rank * per + min(rank, extra)
        return list(range(start, start + per + (1 if rank < extra else 0)))
    raise ValueError("policy must be 'block' or 'round_robin'")


def gather_results(poses, vertices, n_streams: int, policy: str = "block", group=None):
    """Gather every rank's per-stream results to rank 0.

    poses: (S_local, F, 36), vertices: (S_local, F, N, 3) for the streams
    `assign_streams(n_streams, world, rank, policy)`, as torch tensors on the
    process-group device (CUDA for NCCL) or numpy arrays (moved to the
    group's device).  Returns (poses, vertices) of shape (n_streams, ...)
    ordered by global stream id on rank 0, None elsewhere.  Ranks may own
    different stream counts: shards are padded to the largest one for the
    fixed-size gather.
    """
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    p = torch.as_tensor(np.asarray(poses) if not torch.is_tensor(poses) else poses).to(dev, torch.float64)
    v = torch.as_tensor(np.asarray(vertices) if not torch.is_tensor(vertices) else vertices).to(dev, torch.float64)
    smax = max(len(assign_streams(n_streams, world, r, policy)) for r in range(world))
    pad_p = torch.zeros((smax,) + tuple(p.shape[1:]), dtype=p.dtype, device=dev)
    pad_v = torch.zeros((smax,) + tuple(v.shape[1:]), dtype=v.dtype, device=dev)
    pad_p[:p.shape[0]] = p
    pad_v[:v.shape[0]] = v
    # a gather to rank 0 (not an all-gather): only rank 0 consumes results
    out_p = [torch.empty_like(pad_p) for _ in range(world)] if rank == 0 else None
    out_v = [torch.empty_like(pad_v) for _ in range(world)] if rank == 0 else None
    dist.gather(pad_p, out_p, dst=0, group=group)
    dist.gather(pad_v, out_v, dst=0, group=group)
    if rank != 0:
        return None
    P = np.zeros((n_streams,) + tuple(p.shape[1:]))
    V = np.zeros((n_streams,) + tuple(v.shape[1:]))
    for r in range(world):
        ids = assign_streams(n_streams, world, r, policy)
        P[ids] = out_p[r][:len(ids)].cpu().numpy()
        V[ids] = out_v[r][:len(ids)].cpu().numpy()
    return P, V
