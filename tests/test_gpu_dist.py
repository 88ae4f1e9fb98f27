"""Multi-process libsp: world_size 2 over gloo, BOTH ranks drive
libsp on cuda:0 (this pool has one GPU per box; the NCCL path is the same code with CUDA
tensors).  Rank 0 learns with full learning (the inhibition radius adapts, R21), the state --
including the radius in force and the duty cycles -- is broadcast with dist.broadcast_state,
every rank runs batched inference on its contiguous frame shard, and the gathered SDRs (CPU
copies) must equal the single-process oracle for the same global frame indices."""
import os

import numpy as np
import pytest

import oracle as O
import sp_inputs
from tests.helpers import ocfg, gpu_kwargs
from tests.test_dist_gloo import free_port

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOTAL = 46  # 23 inputs per rank (one ragged group each)


def cfg_full():
    return ocfg(input_width=32, input_height=16, num_columns=256, synapses_per_column=24, min_overlap=2,
                winners_set_size=12, inhibition_radius=4, full_learning=True, duty_cycle_period=5)


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    import paper_1608_01966_b200 as P
    from paper_1608_01966_b200 import dist as D
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = cfg_full()
        # rank 1 starts from another seed (and the configured radius): broadcast_state must
        # overwrite the pools, permanences, boosts, duties and the adapted radius
        sp = P.SpatialPooler(**gpu_kwargs(cfg, seed=cfg.seed + rank, max_inputs=64,
                                          flags=P.SP_FLAG_FULL_LEARNING, duty_cycle_period=5))
        if rank == 0:
            frames = torch.from_numpy(sp_inputs.frames(1001, 0, 30, 16, 32, rho=0.5)).cuda()
            sp.compute(frames, learn=True)
        D.broadcast_state(sp, src=0)
        radius = sp.get_learning_state()[2]
        b, e = D.shard_range(TOTAL, rank, world)
        frames = torch.from_numpy(sp_inputs.frames(2002, b, e - b, 16, 32, rho=0.5)).cuda()
        sdr = torch.empty((e - b, sp.sdr_words), dtype=torch.int32, device="cuda")
        cnt = torch.empty((e - b,), dtype=torch.int32, device="cuda")
        sp.compute_into(frames, sdr, cnt)
        gathered = D.gather_sdrs(sdr.cpu())
        q.put((rank, gathered.numpy(), radius, sp.info()["plan"]["path"]))
        sp.close()
    finally:
        dist.destroy_process_group()


def test_two_ranks_libsp_full_learning_broadcast_and_gather():
    import torch.multiprocessing as mp
    import paper_1608_01966_b200 as P
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cfg = cfg_full()
    ora = O.SpatialPoolerOracle(cfg)
    ora.compute(sp_inputs.frames(1001, 0, 30, 16, 32, rho=0.5), learning=True)
    assert ora.radius != cfg.inhibition_radius, "the stream should adapt the radius"
    want = np.stack([O.sdr_words(r.active).view(np.int32)
                     for r in ora.compute(sp_inputs.frames(2002, 0, TOTAL, 16, 32, rho=0.5), False)])
    for rank, gathered, radius, path in res:
        assert radius == ora.radius, f"rank {rank} radius {radius} != {ora.radius}"
        assert path == P.SP_PATH_BATCHED
        assert np.array_equal(gathered, want), f"rank {rank}"
