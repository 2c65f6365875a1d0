"""Model selection host core (no GPU): the W-ensemble clustering, cosine silhouette and Pearson
matrix of the library's C++ host core against the compiled reference
(src/model_selection.cpp:61-314) — bit-identical, since both evaluate the same f64 dot products
in the same order — plus SelectionConfig validation (model_selection.cpp:22-33)."""
import numpy as np
import pytest

import oracle
import paper_2202_09518_b200 as nmf

needs_ref = pytest.mark.skipif(not oracle.ref.available, reason="needs oracle/_ref")


def _same(a, b):
    assert a.min_sil == b["min_sil"] and a.mean_sil == b["mean_sil"]
    assert np.array_equal(a.per_cluster, b["per_cluster"])
    assert np.array_equal(a.medians, b["medians"])
    assert np.array_equal(a.member_cluster, b["member_cluster"])
    assert a.dropped_zero_columns == b["dropped"]


@needs_ref
@pytest.mark.parametrize("runs,m,k", [(2, 10, 1), (3, 40, 2), (6, 50, 5), (16, 64, 8), (5, 33, 16), (4, 30, 20)])
def test_cluster_silhouette_matches_reference(runs, m, k):
    # k <= 16 takes the exact bitmask-DP assignment, k = 20 the greedy one
    rng = np.random.default_rng(runs * 100 + k)
    w = rng.random((runs, m, k))
    _same(nmf.cluster_columns(w), oracle.ref.cluster_silhouette(w))


@needs_ref
def test_ensemble_of_noisy_copies_clusters_perfectly():
    # the structure select_k relies on: runs that are column permutations of one W (plus noise)
    rng = np.random.default_rng(7)
    base = rng.random((80, 6))
    runs = np.stack([base[:, rng.permutation(6)] + 0.01 * rng.random((80, 6)) for _ in range(8)])
    got = nmf.cluster_columns(runs)
    _same(got, oracle.ref.cluster_silhouette(runs))
    assert got.min_sil > 0.9
    for r in range(8):
        assert sorted(got.member_cluster[r].tolist()) == list(range(6))


@needs_ref
def test_zero_columns_are_dropped_like_the_reference():
    rng = np.random.default_rng(3)
    w = rng.random((4, 30, 4))
    w[2, :, 1] = 0.0
    w[3, :, 3] = 0.0
    got = nmf.cluster_columns(w)
    _same(got, oracle.ref.cluster_silhouette(w))
    assert got.dropped_zero_columns == 2 and got.member_cluster[2, 1] == -1


def test_empty_cluster_raises_shape_error():
    w = np.random.default_rng(1).random((3, 20, 3))
    w[0, :, 2] = 0.0  # anchor column gone -> empty cluster -> silhouette refuses
    with pytest.raises(nmf.ShapeError, match="empty cluster"):
        nmf.cluster_columns(w)
    with pytest.raises(nmf.ShapeError):
        nmf.cluster_columns(w[:1])


@needs_ref
def test_pearson_matches_reference_and_rejects_constant_columns():
    rng = np.random.default_rng(2)
    wt, we = rng.random((50, 3)), rng.random((50, 5))
    assert np.array_equal(nmf.pearson_correlation_matrix(wt, we), oracle.ref.pearson(wt, we))
    wt[:, 1] = 0.25
    with pytest.raises(nmf.DataError, match="zero-variance"):
        nmf.pearson_correlation_matrix(wt, we)
    with pytest.raises(nmf.ShapeError):
        nmf.pearson_correlation_matrix(wt[:10], we)


@pytest.mark.parametrize("kw,msg", [(dict(k_min=0), "k_min"), (dict(k_min=3, k_max=2), "k_min"),
                                    (dict(k_max=40), "below min"), (dict(n_perturbations=1), "perturbations"),
                                    (dict(delta=0.0), "delta"), (dict(delta=1.0), "delta"),
                                    (dict(sil_threshold=1.5), "sil_threshold")])
def test_selection_config_validation(kw, msg):
    cfg = nmf.SelectionConfig(**{**dict(k_min=1, k_max=3), **kw})
    with pytest.raises(nmf.ShapeError, match=msg):
        cfg.validate(40, 50)


def test_report_formats():
    rep = nmf.SelectionReport([nmf.KRecord(1, True, 4, 1.0, 1.0, 0.5), nmf.KRecord(2, False, 1)], None, "why")
    csv = rep.to_csv().splitlines()
    assert csv[0] == "k,valid,runs_used,min_silhouette,mean_silhouette,mean_relative_error"
    assert csv[1] == "1,1,4,1,1,0.5" and csv[2] == "2,0,1,0,0,0"
    import json
    j = json.loads(rep.to_json())
    assert j["chosen_k"] == "none" and j["records"][0]["runs_used"] == 4
