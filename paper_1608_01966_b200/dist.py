"""Multi-GPU plumbing: one process per GPU.

Inference frames are independent, so they are sharded across ranks by
contiguous global frame ranges with no data-path collective.  The SP state is
replicated with one broadcast at setup, and the winner SDRs of every step are
all-gathered to every rank (north_star: "NCCL over NVLink only for gathering
winner SDRs to the classifier").  Learning is a sequential recurrence over
frames and stays on one GPU ("replicas only").

Works with any torch.distributed backend: NCCL with CUDA tensors on the GPU
box, gloo with CPU tensors in the CPU tests.
"""
from __future__ import annotations

import numpy as np


def shard_range(total: int, rank: int, world: int):
    """Contiguous [begin, end) of ``total`` frames owned by ``rank`` (balanced, in order)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    return total * rank // world, total * (rank + 1) // world


def broadcast_arrays(arrays, src: int, device=None):
    """Broadcasts a list of numpy arrays (shapes/dtypes known on every rank) from ``src``."""
    import torch
    import torch.distributed as dist
    out = []
    for a in arrays:
        t = torch.from_numpy(np.ascontiguousarray(a))
        if device is not None:
            t = t.to(device)
        if t.dtype == torch.uint32:  # NCCL/gloo have no uint32: move the bits as int32
            t = t.view(torch.int32)
        dist.broadcast(t, src=src)
        out.append(t.cpu().numpy().view(a.dtype).reshape(a.shape))
    return out


def broadcast_state(sp, src: int = 0, device=None):
    """Replicates the learned state of rank ``src``'s SpatialPooler to every rank.

    Besides the synapses and boosts this carries the learning state (duty cycles and the
    inhibition radius in force): with full learning the radius adapts (R21) and the
    batched inference reads it, so a replica left at the configured radius would pick
    different winners than one GPU does."""
    idx, perm, boost = sp.get_state()
    adc, odc, radius, _ = sp.get_learning_state()
    r = np.array([radius], dtype=np.int64)
    idx, perm, boost, adc, odc, r = broadcast_arrays([idx, perm, boost, adc, odc, r], src, device)
    import torch.distributed as dist
    if dist.get_rank() != src:
        sp.set_state(idx, perm, boost)
        sp.set_learning_state(adc, odc, int(r[0]))
    return idx, perm, boost


def gather_sdrs(local_sdr, out=None):
    """All-gathers the [n_local, words] int32 SDR tensor of every rank -> [n_local*world, words].

    Shards must be equal-sized (weak scaling, or total divisible by world)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size()
    if out is None:
        out = torch.empty((local_sdr.shape[0] * world, local_sdr.shape[1]), dtype=local_sdr.dtype,
                          device=local_sdr.device)
    dist.all_gather_into_tensor(out, local_sdr.contiguous())
    return out


def gather_histograms(local_hist, out=None):
    """All-gathers per-video SDR histograms (NEXT-4) of every rank: [V_local, C] -> [V_local*world, C].

    Videos are sharded whole (each rank holds complete videos, equal counts per rank), so the
    per-video features replace the per-frame SDR gather on the way to the classifier rank."""
    return gather_sdrs(local_hist, out)
