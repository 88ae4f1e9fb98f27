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
