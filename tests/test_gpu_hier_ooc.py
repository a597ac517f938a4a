"""GPU parity of rw_hier_segment_ooc (SURVEY §8(f) f1 out of core: host volume / labels /
output, brick pool + page tables instead of dense level fields; P:105, P:109-111, P:151,
reading R31) against oracle/hier_oracle.py on ragged non-cubic volumes, and bit-for-bit
agreement with the in-HBM driver rw_hier_segment on cubic s 2^k volumes."""
import numpy as np
import pytest
import torch

import paper_2103_09564_b200 as rwb
from oracle import hier_oracle as ho
from paper_2103_09564_b200._lib import RWError
from gpu_helpers import dev
from test_hier_oracle import small_volume
from test_hier_ragged_pins import _ragged_volume

pytestmark = pytest.mark.gpu

P_TOL = 1e-4   # as test_gpu_hier.py: GPU tol 1e-7 vs oracle 1e-10, errors through <= 4 levels


def _check_vs_oracle(vol, seeds, **kw):
    prob, lab, st = rwb.hier_segment_ooc(vol, seeds, tol=1e-7, max_iter=20000, **kw)
    ref = ho.hier_segment(vol, seeds, tol=1e-10, **kw)
    assert st["levels"] == len(ref["stats"])
    for l, rs in enumerate(ref["stats"]):
        assert st["solved"][l] == rs["solved"], (l, st, ref["stats"])
        assert st["pruned_hom"][l] == rs["pruned_hom"] and st["pruned_dt"][l] == rs["pruned_dt"]
        assert st["conflict"][l] == rs["conflict"]
    d = np.abs(prob.astype(np.float64) - ref["prob"])
    assert d.max() <= P_TOL, d.max()
    sure = np.abs(ref["prob"] - 0.5) > 1e-3
    assert np.array_equal(lab[sure], (ref["prob"] > 0.5)[sure])
    assert np.array_equal(lab, (prob > 0.5).astype(np.uint8))     # labels = p > 0.5 (R10)
    return prob, st


@pytest.mark.parametrize("shape,prune", [((40, 56, 72), False), ((40, 56, 72), True),
                                         ((36, 64, 48), True), ((24, 40, 72), False)])
def test_ooc_ragged_matches_oracle(shape, prune):
    """Ragged, non-cubic volumes, s = 16, e = 1.25: smaller border bricks on every level,
    windows narrower than s_e at the coarse levels, x sides padded to a multiple of 4 (root
    9 -> 12, level 2 18 -> 20)."""
    vol, seeds = _ragged_volume(shape, 1, 150)
    _, st = _check_vs_oracle(vol, seeds, s=16, e=1.25, beta=100.0, prune=prune)
    assert st["pool_used"] >= sum(st["solved"])


@pytest.mark.parametrize("D,s,e,prune", [(64, 16, 1.25, True), (64, 16, 1.25, False),
                                         (32, 8, 1.5, True)])
def test_ooc_cubic_matches_oracle(D, s, e, prune):
    vol, seeds = small_volume(D, seed=D + s)
    _check_vs_oracle(vol, seeds, s=s, e=e, beta=50.0, prune=prune)


@pytest.mark.parametrize("D,s,prune", [(128, 16, True), (256, 32, True), (256, 32, False),
                                       (512, 32, True)])
def test_ooc_bitwise_equals_in_hbm_driver(D, s, prune):
    """Cubic s 2^k: the page-table field (materialised upsamples, pool) reproduces the dense
    field pyramid of rw_hier_segment bit for bit (same samples, same solves; the resident
    solver for s_e = 40).  D = 512: the level-0 upsample of the in-HBM driver is the z-walk
    kernel (k_upsample_walk, levels of side >= 512), checked here against the per-sample
    form (hier::sample in k_ooc_materialize / k_ooc_out)."""
    vol, seeds = small_volume(D, seed=3)
    kw = dict(s=s, e=1.25, beta=50.0, tol=1e-6, prune=prune)
    ref, st_ref, _ = rwb.hier_segment(dev(vol), dev(seeds), **kw)
    torch.cuda.synchronize()
    prob, lab, st = rwb.hier_segment_ooc(vol, seeds, **kw)
    assert st["solved"] == st_ref["solved"] and st["iters"] == st_ref["iters"]
    assert np.array_equal(prob, ref.cpu().numpy())
    assert np.array_equal(lab, (prob > 0.5).astype(np.uint8))


def test_ooc_labels_only_and_single_brick():
    """Labels without the fp32 output; a volume that is one brick (root = level 0, windows
    from host memory) equals rw_solve_bricks on the whole volume."""
    vol, seeds = _ragged_volume((12, 16, 20), 2, 10)
    prob, lab, st = rwb.hier_segment_ooc(vol, seeds, s=32, e=1.25, beta=50.0, tol=1e-7)
    assert st["levels"] == 1 and st["solved"] == [1]
    fixed, val = ho.seeds_from_bits(ho.seed_bits(seeds))
    out = rwb.solve_bricks(dev(fixed.astype(np.uint8)), dev(val.astype(np.float32)),
                           vol=dev(vol), beta=50.0, tol=1e-7)
    torch.cuda.synchronize()
    assert np.abs(prob - out["prob"][0, 0].cpu().numpy()).max() <= 1e-5
    p2, l2, _ = rwb.hier_segment_ooc(vol, seeds, s=32, e=1.25, beta=50.0, tol=1e-7,
                                     want_prob=False)
    assert p2 is None and np.array_equal(l2, lab)


def test_ooc_page_locked_buffers_are_bitwise_the_pageable_run():
    """Page-locked volume / seeds (cudaHostRegister) and pinned outputs take the direct copy-engine
    path (no staging through the queue's host slots), with a reused queue + workspace: the same
    bits as the pageable call, twice in a row (slot reuse), with and without the fp32 field."""
    vol, seeds = _ragged_volume((72, 88, 104), 2, 21)
    kw = dict(s=16, e=1.25, beta=50.0, tol=1e-6)
    prob, lab, st = rwb.hier_segment_ooc(vol, seeds, **kw)
    q, ws, pool = rwb.hier_ooc_alloc(vol.shape, vol.dtype, s=16)
    op, ol = rwb.pinned_empty(vol.shape, np.float32), rwb.pinned_empty(vol.shape, np.uint8)
    try:
        with rwb.host_register(vol), rwb.host_register(seeds):
            for rep in range(2):
                op.fill(-1.0), ol.fill(255)
                p2, l2, st2 = rwb.hier_segment_ooc(vol, seeds, queue=q, workspace=ws, pool_bricks=pool,
                                                   out_prob=op, out_labels=ol, **kw)
                assert p2 is op and l2 is ol
                assert st2["solved"] == st["solved"] and st2["iters"] == st["iters"]
                assert np.array_equal(op, prob) and np.array_equal(ol, lab)
            ol.fill(255)
            p3, l3, _ = rwb.hier_segment_ooc(vol, seeds, queue=q, workspace=ws, pool_bricks=pool,
                                             want_prob=False, out_labels=ol, **kw)
            assert p3 is None and np.array_equal(ol, lab)
        with pytest.raises(ValueError):
            rwb.hier_segment_ooc(vol, seeds, out_labels=np.empty(vol.shape, np.float32), **kw)
    finally:
        q.close()


@pytest.mark.parametrize("limit", ["0", "3"])
def test_ooc_sparse_seed_upload_equals_dense(limit, monkeypatch):
    """The pyramid phase uploads only the non-zero 4 KiB segments of each slab's seed bytes
    (the rest is a device memset); with the segment limit at 0 (always dense) or 3 (slabs with
    more seeded segments fall back to the dense copy) the run gives the same bits, for
    pageable and page-locked seeds."""
    vol, seeds = _ragged_volume((72, 88, 104), 4, 40)
    kw = dict(s=16, e=1.25, beta=50.0, tol=1e-6)
    prob, lab, st = rwb.hier_segment_ooc(vol, seeds, **kw)
    monkeypatch.setenv("RW_OOC_SEED_SEGS", limit)
    p2, l2, st2 = rwb.hier_segment_ooc(vol, seeds, **kw)
    assert st2["solved"] == st["solved"] and st2["iters"] == st["iters"]
    assert np.array_equal(p2, prob) and np.array_equal(l2, lab)
    with rwb.host_register(vol), rwb.host_register(seeds):
        p3, l3, _ = rwb.hier_segment_ooc(vol, seeds, **kw)
    assert np.array_equal(p3, prob) and np.array_equal(l3, lab)


def test_ooc_pool_full_is_an_error():
    vol, seeds = small_volume(64, seed=5)
    with pytest.raises(RWError, match="RW_ENOMEM"):
        rwb.hier_segment_ooc(vol, seeds, s=16, e=1.25, beta=50.0, prune=False, pool_bricks=4)


def _ragged_classes(shape, seed, nseed):
    """Three-class seeds on a ragged volume: the blob seeds are class 1, the outside seeds
    class 2 (lower z half) or 3 (upper z half)."""
    vol, seeds = _ragged_volume(shape, seed, nseed)
    lab = seeds.copy()
    z = np.arange(shape[0])[:, None, None]
    lab[(seeds == 2) & (z >= shape[0] // 2)] = 3
    return vol, lab


@pytest.mark.parametrize("shape,prune", [((40, 56, 72), True), ((36, 64, 48), False)])
def test_ooc_labels_ragged_match_oracle(shape, prune):
    """rw_hier_segment_labels_ooc on ragged non-cubic volumes: K = 3 one-vs-rest
    out-of-core runs (class seeds remapped on the device after the H2D copy, running maximum
    merged on the host) against the oracle's K explicit runs: pruning decisions identical,
    best = the winning class's probability within P_TOL, labels equal wherever the oracle's
    top two classes differ by more than 1e-3 (reading R18)."""
    vol, lab = _ragged_classes(shape, 2, 120)
    best, got, st = rwb.hier_segment_labels_ooc(vol, lab, 3, s=16, e=1.25, beta=100.0, tol=1e-7,
                                                max_iter=20000, prune=prune)
    ref = ho.hier_segment_labels(vol, lab, 3, s=16, e=1.25, beta=100.0, tol=1e-10, prune=prune)
    for k in range(3):
        for l, rs in enumerate(ref["stats"][k]):
            g = st[k]
            assert g["solved"][l] == rs["solved"] and g["pruned_hom"][l] == rs["pruned_hom"]
            assert g["pruned_dt"][l] == 0 and g["conflict"][l] == rs["conflict"]
    assert got.min() >= 1 and got.max() <= 3
    assert np.abs(best.astype(np.float64) - ref["prob"].max(0)).max() <= P_TOL
    srt = np.sort(ref["prob"], axis=0)
    sure = srt[-1] - srt[-2] > 1e-3
    assert sure.mean() > 0.9
    assert np.array_equal(got[sure], ref["labels"][sure])


@pytest.mark.parametrize("D,s,prune", [(128, 16, True), (64, 16, False)])
def test_ooc_labels_bitwise_equal_in_hbm_driver(D, s, prune):
    """Cubic s 2^k: best / labels equal rw_hier_segment_labels' bit for bit, and the merged
    best is the maximum over the K binary out-of-core runs on the one-vs-rest seeds."""
    from test_hier_oracle import multi_volume
    vol, lab = multi_volume(D, seed=7)
    kw = dict(s=s, e=1.25, beta=50.0, tol=1e-6, prune=prune)
    ref = rwb.hier_segment_labels(dev(vol), dev(lab), 3, **kw)
    torch.cuda.synchronize()
    best, got, st = rwb.hier_segment_labels_ooc(vol, lab, 3, **kw)
    assert np.array_equal(best, ref["best"].cpu().numpy())
    assert np.array_equal(got, ref["labels"].cpu().numpy())
    for k in range(3):
        assert st[k]["solved"] == ref["stats"][k]["solved"]
    fields = []
    for k in range(1, 4):
        seeds = np.where(lab == k, 1, np.where(lab > 0, 2, 0)).astype(np.uint8)
        p, _, _ = rwb.hier_segment_ooc(vol, seeds, t_bin=-1.0, **kw)
        fields.append(p)
    fields = np.asarray(fields)
    assert np.array_equal(best, fields.max(0))
    assert np.array_equal(got, (np.argmax(fields, 0) + 1).astype(np.uint8))   # ties -> lowest id


def test_ooc_labels_rejects_bad_arguments():
    from test_hier_oracle import multi_volume
    vol, lab = multi_volume(32, seed=1)
    with pytest.raises(RWError, match="K must be in 2..255"):
        rwb.hier_segment_labels_ooc(vol, lab, 1, s=8, e=1.5)
    with pytest.raises(ValueError):
        rwb.hier_segment_labels_ooc(vol, lab[:-1], 3, s=8, e=1.5)
