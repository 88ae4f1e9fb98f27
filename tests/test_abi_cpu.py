"""CPU-only checks of the C-ABI library: it loads, exports every symbol the
headers declare, and its host logic (validation, seeded init, planner) is right.
No compute calls are made here (no GPU in the CI container)."""
import os
import re

import numpy as np
import pytest

import oracle as O
import paper_1608_01966_b200 as P
from paper_1608_01966_b200 import build as B

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def built():
    B.build()


def declared_symbols():
    names = set()
    for h in sorted(os.listdir(os.path.join(ROOT, "include"))):
        txt = open(os.path.join(ROOT, "include", h)).read()
        names |= set(re.findall(r"^\s*(?:sp_status|const char\*)\s+(sp_\w+)\s*\(", txt, re.M))
    return names


def test_library_exports_every_declared_symbol():
    L = P.lib()
    decl = declared_symbols()
    assert decl == set(P.ABI_SYMBOLS), decl ^ set(P.ABI_SYMBOLS)
    for name in decl:
        assert hasattr(L, name), name
    assert b"sm_100a" in L.sp_version()


def test_library_is_sm100a_only():
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump --list-elf {P.sp.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out.replace("sm_100a", "")), out


@pytest.mark.parametrize("kw", [
    dict(input_width=8, input_height=8, num_columns=128, synapses_per_column=16),
    dict(input_width=960, input_height=540, num_columns=40, synapses_per_column=256, seed=7),
    dict(input_width=48, input_height=37, num_columns=100, synapses_per_column=1776, seed=3),
    dict(input_width=960, input_height=540, patch_width=32, patch_height=30, num_columns=50,
         synapses_per_column=960, seed=11),
])
def test_library_init_equals_oracle_init(kw):
    # the C library and the oracle implement R8 independently; they must agree
    got = P.init_pools_host(**kw)
    okw = {k: v for k, v in kw.items()}
    want, _, _ = O.init_pools(O.OracleConfig(**okw))
    assert np.array_equal(got.astype(np.int64), want)


@pytest.mark.parametrize("bad,msg", [
    (dict(synapses_per_column=100), "S:50"),
    (dict(min_overlap=20), "min_overlap"),
    (dict(winners_set_size=200), "winners_set_size"),
    (dict(winners_set_size=0), "winners_set_size"),
    (dict(perm_increment=1.5), "perm_increment"),
    (dict(connected_threshold=-0.1), "connected_threshold"),
    (dict(patch_width=3, patch_height=3), "divide"),
    (dict(patch_width=4, patch_height=0), "both"),
    (dict(num_columns=0), "num_columns"),
    (dict(max_inputs=0), "max_inputs"),
])
def test_config_validation(bad, msg):
    kw = dict(input_width=8, input_height=8, num_columns=128, synapses_per_column=16, min_overlap=2,
              winners_set_size=8)
    kw.update(bad)
    with pytest.raises(P.SpError) as ei:
        P.plan(1, **kw)
    assert ei.value.status == P.SP_E_CONFIG and msg in ei.value.message


def test_plan_headline_is_batched_and_fits_one_wave():
    pl = P.plan(4096, input_width=960, input_height=540, num_columns=1024, synapses_per_column=256,
                min_overlap=4, winners_set_size=40)
    assert pl["path"] == P.SP_PATH_BATCHED and pl["reason"] == 0
    assert pl["ctas"] <= 148 and pl["groups"] * 32 >= 4096
    assert pl["smem_bytes"] <= 232448
    assert pl["num_windows"] * pl["window_bits"] >= 518400


def test_plan_small_batches_split_windows_over_clusters():
    # 512 frames (8-GPU shard of 4096): a cluster of CTAs shares each group
    pl = P.plan(512, input_width=960, input_height=540, num_columns=1024, synapses_per_column=256)
    assert pl["cluster"] > 1 and pl["ctas"] <= 148


def test_plan_patch_mode_uses_the_patch_kernel():
    # 960x540 in 32x30 tiles: 30 tiles per tile-row -> one group per tile-row (NEXT-2)
    pl = P.plan(4, input_width=960, input_height=540, patch_width=32, patch_height=30,
                num_columns=1024, synapses_per_column=256)
    assert pl["path"] == P.SP_PATH_BATCHED and pl["groups"] == 4 * 18 and pl["num_windows"] == 1


@pytest.mark.parametrize("kw,reason", [
    (dict(input_width=960, input_height=540, patch_width=16, patch_height=30), 2),
    (dict(input_width=37, input_height=5), 4),
    (dict(input_width=960, input_height=540, num_columns=16384, synapses_per_column=512), 8),
    (dict(input_width=960, input_height=540, force_path=P.SP_PATH_PER_INPUT), 32),
])
def test_plan_falls_back_to_per_input_path(kw, reason):
    base = dict(num_columns=1024, synapses_per_column=64)
    base.update(kw)
    pl = P.plan(4, **base)
    assert pl["path"] == P.SP_PATH_PER_INPUT and pl["reason"] & reason


def test_create_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(P.SpError) as ei:
        P.SpatialPooler(input_width=8, input_height=8, num_columns=128, synapses_per_column=16)
    assert ei.value.status == P.SP_E_CUDA


def test_encoder_create_without_gpu_fails_loudly():
    # no CPU fallback for the encoder either: creation needs a CUDA device (CPU box: SP_E_CUDA)
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(P.SpError) as e:
        P.Encoder()
    assert e.value.status == P.SP_E_CUDA


@pytest.mark.parametrize("n", [1, 7, 33, 100, 256, 512, 777, 1024, 2048, 4095, 4096, 10000])
@pytest.mark.parametrize("sm_count", [148, 132])
def test_plan_groups_of_exact_rows(n, sm_count):
    """Whole-frame plans: groups of exactly R <= 32 inputs (the TMA box rows), the
    last one shorter; stages of R KiB in the 140 KiB ring (4..8); a global split never needs
    more CTAs than SMs (cooperative launch), a cluster never more than 16 CTAs."""
    pl = P.plan(n, sm_count=sm_count, input_width=960, input_height=540, num_columns=1024,
                synapses_per_column=256)
    R, G, K = pl["group_inputs"], pl["groups"], pl["cluster"]
    assert pl["path"] == P.SP_PATH_BATCHED and 1 <= R <= 32
    assert G == -(-n // R) and pl["ctas"] == G * K
    assert 4 <= pl["stages"] <= 8 and pl["stages"] * R * 1024 <= 140 * 1024
    if pl["global_split"]:
        assert 2 <= K <= 16 and pl["ctas"] <= sm_count
    else:
        assert 1 <= K <= 8


def test_plan_headline_groups_of_28():
    pl = P.plan(4096, sm_count=148, input_width=960, input_height=540, num_columns=1024,
                synapses_per_column=256, min_overlap=4, winners_set_size=40)
    assert (pl["groups"], pl["group_inputs"], pl["cluster"], pl["stages"], pl["global_split"]) == (147, 28, 1, 5, 0)
