"""Host logic of the multi-GPU path that needs no GPU: the exact seismogram
merge of a slab decomposition (dist.merge_seismogram) and the FDW_DEVICES
parser shared with the C++ drop-in."""
import numpy as np

from paper_2201_05278_b200.dist import merge_seismogram
from paper_2201_05278_b200.multi import devices_from_env


def _sequential(products):
    acc = 0.0
    for p in products:
        acc += p
    return acc


def test_merge_reproduces_one_sequential_accumulation():
    rng = np.random.default_rng(1)
    rows, n_rec = 7, 5
    # receiver 1 straddles ranks 0 / 1 (entries 0..5 on rank 0, 6..11 on rank 1), receiver 3
    # straddles ranks 1 / 2; the others live on one rank (partials)
    prod = {1: rng.standard_normal((rows, 12)) * 10.0 ** rng.integers(-8, 8, 12),
            3: rng.standard_normal((rows, 9)) * 10.0 ** rng.integers(-8, 8, 9)}
    partials = [np.zeros((rows, n_rec)) for _ in range(3)]
    for r, rec in ((0, 0), (1, 2), (2, 4)):
        partials[r][:, rec] = rng.standard_normal(rows)
    splits = []
    for r in range(3):
        recs, ents, cols = [], [], []
        for p, (lo, hi) in ((1, {0: (0, 6), 1: (6, 12)}.get(r, (0, 0))), (3, {1: (0, 4), 2: (4, 9)}.get(r, (0, 0)))):
            for e in range(lo, hi):
                recs.append(p)
                ents.append(e)
                cols.append(prod[p][:, e])
        # a rank lists its slots in any order: the merge orders them by entry
        order = rng.permutation(len(recs)) if recs else []
        splits.append((np.array(recs, np.uint64)[order] if recs else np.zeros(0, np.uint64),
                       np.array(ents, np.uint64)[order] if recs else np.zeros(0, np.uint64),
                       np.stack(cols, axis=1)[:, order] if recs else np.zeros((rows, 0))))
    out = merge_seismogram([p.reshape(-1) for p in partials], splits, n_rec).reshape(rows, n_rec)
    for row in range(rows):
        for p in (1, 3):
            assert out[row, p] == _sequential(prod[p][row])  # bit for bit, not approximately
        assert out[row, 0] == partials[0][row, 0] and out[row, 4] == partials[2][row, 4]


def test_merge_all_negative_zero_products_give_plus_zero():
    splits = [(np.array([0], np.uint64), np.array([0], np.uint64), np.full((2, 1), -0.0)),
              (np.array([0], np.uint64), np.array([1], np.uint64), np.full((2, 1), -0.0))]
    out = merge_seismogram([np.zeros(2), np.zeros(2)], splits, 1)
    assert np.all(out == 0) and not np.any(np.signbit(out))  # 0.0 + (-0.0) = +0.0, as the reference


def test_devices_from_env(monkeypatch):
    monkeypatch.setenv("FDW_DEVICES", "0-3")
    assert devices_from_env() == [0, 1, 2, 3]
    monkeypatch.setenv("FDW_DEVICES", "0,0, 2")
    assert devices_from_env() == [0, 0, 2]
    monkeypatch.delenv("FDW_DEVICES")
    assert devices_from_env() == []
