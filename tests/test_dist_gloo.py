"""N > 1 host logic on CPU: world_size-2 gloo process group (the GPU box runs the
same code with NCCL).  Frames are sharded by contiguous global ranges, the SP
state is broadcast once, and the gathered SDRs must equal the single-process
result for the same global frame indices."""
import os
import socket

import numpy as np
import pytest

import oracle as O
import sp_inputs
from paper_1608_01966_b200 import dist as D


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, total, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = O.OracleConfig(input_width=8, input_height=8, num_columns=128, synapses_per_column=16,
                             min_overlap=2, winners_set_size=8, seed=42)
        # state: rank 0 owns a learned state; the others start from garbage and receive it
        if rank == 0:
            ora = O.SpatialPoolerOracle(cfg)
            ora.compute(sp_inputs.frames(1001, 0, 10, 8, 8), learning=True)
            arrays = [ora.idx.astype(np.uint32), ora.perm, ora.boost]
        else:
            arrays = [np.zeros((128, 16), np.uint32), np.zeros((128, 16), np.float32),
                      np.zeros(128, np.float32)]
        idx, perm, boost = D.broadcast_arrays(arrays, src=0)
        ora = O.SpatialPoolerOracle(cfg, (idx, perm, boost))
        b, e = D.shard_range(total, rank, world)
        frames = sp_inputs.frames(2002, b, e - b, 8, 8)
        local = np.stack([O.sdr_words(r.active).view(np.int32) for r in ora.compute(frames, False)])
        out = D.gather_sdrs(torch.from_numpy(local))
        # per-video histograms of this rank's whole videos (3 frames each), gathered (NEXT-4)
        act = np.stack([r.active for r in ora.compute(frames, False)])
        _, hist = O.sdr_histograms(act, np.arange(0, e - b + 1, 3))
        hist_all = D.gather_histograms(torch.from_numpy(hist))
        q.put((rank, out.numpy(), idx, perm, hist_all.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_inference_gathers_identical_sdrs(world):
    import torch.multiprocessing as mp
    total = 12
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, total, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort(key=lambda t: t[0])
    # single-process reference with the same learned state and global frame indices
    cfg = O.OracleConfig(input_width=8, input_height=8, num_columns=128, synapses_per_column=16,
                         min_overlap=2, winners_set_size=8, seed=42)
    ora = O.SpatialPoolerOracle(cfg)
    ora.compute(sp_inputs.frames(1001, 0, 10, 8, 8), learning=True)
    want = np.stack([O.sdr_words(r.active).view(np.int32)
                     for r in ora.compute(sp_inputs.frames(2002, 0, total, 8, 8), False)])
    act = np.stack([r.active for r in ora.compute(sp_inputs.frames(2002, 0, total, 8, 8), False)])
    _, want_hist = O.sdr_histograms(act, np.arange(0, total + 1, 3))
    for rank, gathered, idx, perm, hist_all in res:
        assert np.array_equal(gathered, want), f"rank {rank}"
        assert np.array_equal(hist_all, want_hist), f"rank {rank} histograms"
        assert np.array_equal(idx.astype(np.int64), ora.idx) and np.array_equal(perm, ora.perm)


def test_shard_range_partitions():
    for total in (0, 1, 7, 4096, 4097):
        for world in (1, 2, 3, 8):
            spans = [D.shard_range(total, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [e - b for b, e in spans]
            assert max(sizes) - min(sizes) <= 1
