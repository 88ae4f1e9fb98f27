"""Shared test helpers: seeded states and oracle/GPU comparison utilities.

Only tests import this.  State arrays are produced by the oracle's init plus
seeded perturbations from ``sp_inputs``-style hashing (never from the CUDA path).
"""
import numpy as np

import oracle as O
import sp_inputs

# permanence values around tau = 0.2 reachable by the fp32 +/-0.1 walk (DESIGN R3)
NEAR_TAU = np.array([0.0, 0.11, 0.19999993, 0.2, 0.20000002, 0.21, 0.31, 1.0], np.float32)


def ocfg(**kw):
    base = dict(input_width=8, input_height=8, num_columns=128, synapses_per_column=16,
                min_overlap=2, winners_set_size=8, inhibition_radius=0, seed=42)
    base.update(kw)
    return O.OracleConfig(**base)


def gpu_kwargs(cfg: O.OracleConfig, **extra):
    d = dict(input_width=cfg.input_width, input_height=cfg.input_height,
             patch_width=cfg.patch_width, patch_height=cfg.patch_height,
             num_columns=cfg.num_columns, synapses_per_column=cfg.synapses_per_column,
             min_overlap=cfg.min_overlap, winners_set_size=cfg.winners_set_size,
             inhibition_radius=cfg.inhibition_radius, perm_increment=cfg.perm_increment,
             perm_decrement=cfg.perm_decrement, initial_permanence=cfg.initial_permanence,
             connected_threshold=cfg.connected_threshold, seed=cfg.seed)
    d.update(extra)
    return d


def perturbed_state(cfg: O.OracleConfig, seed: int = 5, boost_seed: int = 7, boost_hi: float = 2.0):
    """Oracle init pools + seeded permanences near tau + seeded boosts (C11)."""
    idx, _, _ = O.init_pools(cfg)
    rng = np.random.default_rng(seed)
    perm = rng.choice(NEAR_TAU, size=idx.shape, p=[.05, .1, .1, .15, .15, .25, .1, .1]).astype(np.float32)
    boost = sp_inputs.boosts(boost_seed, cfg.num_columns, 1.0, boost_hi)
    return idx, perm, boost


def sdr_of(active):
    return O.sdr_words(active).view(np.int32)


# --------------------------------------------------------------------------- #
# oracle on many frames: a fork Pool over frame chunks (inference inputs are independent)
# --------------------------------------------------------------------------- #
_POOL = None


def _pool_job(job):
    first, count, stride = job
    cfg, state, seed, rho = _POOL
    ora = O.SpatialPoolerOracle(cfg, state)
    out = []
    for j in range(count):
        f = first + j * stride
        x = O.encode(sp_inputs.frames(seed, f, 1, cfg.input_height, cfg.input_width, rho=rho), cfg)
        for xi in x:
            r = ora.step(xi, False)
            out.append((f, sdr_of(r.active), int(r.active.sum())))
    return out


def oracle_infer_frames(cfg, state, seed, frame_ids, rho=0.5, processes=None):
    """Oracle inference on frames ``frame_ids`` of the seeded stream ``seed`` (regenerated on the
    host from sp_inputs), split over a fork Pool: {frame: [(sdr int32 words, count) per input]}."""
    import multiprocessing as mp
    import os
    global _POOL
    _POOL = (cfg, state, seed, rho)
    ids = list(frame_ids)
    n = processes or max(1, min(len(os.sched_getaffinity(0)), 64))
    chunks = [ids[i::n] for i in range(n)]
    jobs = []
    for ch in chunks:
        if not ch:
            continue
        stride = ch[1] - ch[0] if len(ch) > 1 else 1
        assert all(ch[i] == ch[0] + i * stride for i in range(len(ch)))
        jobs.append((ch[0], len(ch), stride))
    with mp.get_context("fork").Pool(len(jobs)) as pool:
        parts = pool.map(_pool_job, jobs, chunksize=1)
    res = {}
    for part in parts:
        for f, s, c in part:
            res.setdefault(f, []).append((s, c))
    return res
