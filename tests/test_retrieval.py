"""Retrieval top-K against the reference DescriptorIndex.

Goldens (tests/golden/retrieval.npz, ``make_golden.retrieval_vectors``): the
reference's topk on two random indexes (D=16, D=256) whose ids are not in
insertion order, with exact ties (identical directions) at the top and a
k > size case.  The host mirror must match bit for bit; the GPU batch path
must return the same ids with similarities within a few ulp.
"""

import numpy as np
import pytest


def _index(d, tag, n=None):
    from paper_2601_04185_b200.retrieval import DescriptorIndex
    vecs, ids = d[f"{tag}_vecs"], d[f"{tag}_ids"]
    n = vecs.shape[0] if n is None else n
    idx = DescriptorIndex(vecs.shape[1])
    for i in range(n):
        idx.add(f"e{ids[i]:04d}", vecs[i])
    return idx, [f"e{i:04d}" for i in ids]


def test_host_topk_matches_reference(golden):
    d = golden("retrieval")
    for tag in ("a", "b"):
        idx, names = _index(d, tag)
        for qi, q in enumerate(d[f"{tag}_qs"]):
            r = idx.topk(q, 12)
            assert [names.index(e) for e, _ in r] == list(d[f"{tag}_top"][qi])
            assert np.array_equal(np.array([s for _, s in r]), d[f"{tag}_sims"][qi])
        small, _ = _index(d, tag, 5)
        assert [names.index(e) for e, _ in small.topk(d[f"{tag}_qs"][1], 12)] == list(d[f"{tag}_small_top"])


def test_host_topk_errors():
    from paper_2601_04185_b200.retrieval import DescriptorIndex
    idx = DescriptorIndex(4).add("a", np.ones(4))
    with pytest.raises(ValueError):
        idx.topk(np.zeros(4), 1)
    with pytest.raises(ValueError):
        idx.topk(np.ones(4), 0)
    with pytest.raises(ValueError):
        idx.add("a", np.ones(4))
    with pytest.raises(ValueError):
        idx.add("b", np.zeros(4))


@pytest.mark.gpu
def test_gpu_topk_batch_matches_reference(golden):
    d = golden("retrieval")
    for tag in ("a", "b"):
        idx, names = _index(d, tag)
        ids, sims = idx.topk_batch(d[f"{tag}_qs"], 12)
        for qi in range(len(ids)):
            assert [names.index(e) for e in ids[qi]] == list(d[f"{tag}_top"][qi]), (tag, qi)
        assert np.abs(sims - d[f"{tag}_sims"]).max() < 1e-14
        small, _ = _index(d, tag, 5)
        sid, ss = small.topk_batch(d[f"{tag}_qs"][1:2], 12)
        assert [names.index(e) for e in sid[0]] == list(d[f"{tag}_small_top"]) and ss.shape == (1, 5)


@pytest.mark.gpu
def test_gpu_topk_batch_errors():
    from paper_2601_04185_b200.retrieval import DescriptorIndex
    idx = DescriptorIndex(4).add("a", np.ones(4)).add("b", np.arange(4.0) + 1)
    with pytest.raises(ValueError, match="non-zero and finite"):
        idx.topk_batch(np.zeros((2, 4)), 1)
    with pytest.raises(ValueError):
        idx.topk_batch(np.ones((2, 4)), 0)
    with pytest.raises(ValueError):
        idx.topk_batch(np.ones((2, 5)), 1)
    ids, _ = idx.topk_batch(np.ones((3, 4)), 2)
    assert ids == [["a", "b"]] * 3


@pytest.mark.gpu
def test_gpu_retrieval_localize_batch_equals_host(golden):
    """localize_batch with GPU ranking == host ranking on the reference scene (k_loc < entries)."""
    from paper_2601_04185_b200.localizer import localize_batch
    from paper_2601_04185_b200.posest import RansacConfig
    from scene_io import unpack_scene
    vmap, jobs = unpack_scene(golden("lift"))
    assert all(j.k_loc < len(vmap.entries) for j in jobs)
    cfg = RansacConfig(seed=5)
    a = localize_batch(jobs, vmap, cfg, seeds=[100 + j for j in range(len(jobs))], depth_cache={})
    b = localize_batch(jobs, vmap, cfg, seeds=[100 + j for j in range(len(jobs))], depth_cache={}, retrieval="gpu")
    for x, y in zip(a, b):
        assert np.array_equal(x.pose.q, y.pose.q) and np.array_equal(x.pose.t, y.pose.t)
        assert np.array_equal(x.inlier_flags, y.inlier_flags) and x.iterations == y.iterations
