"""Standalone reduction entry points against the reference's own outputs
(tests/golden/make_golden_misc.py): commodity_sums / edge_loads /
edge_loads_from_pairs (model.py:297-319), det_diff_norm (_reduce.py:118-128)
and score_paths (projection.py:22-32).  Bitwise.

CPU: the oracle (the checker) against the fixtures.
GPU (-m gpu): the C-ABI entry points pf_commodity_sums / pf_edge_loads /
pf_edge_loads_from_pairs / pf_det_diff_norm / pf_score_paths against the fixtures.
"""

import functools
import os

import numpy as np
import pytest

import golden_io as G

TAGS = G.SMALL + ("cfg1_v0.3",)


@functools.lru_cache(maxsize=1)
def misc():
    return dict(np.load(os.path.join(G.GOLDEN, "golden_misc.npz")))


def _lengths():
    return sorted({int(k.split("/")[1]) for k in misc() if k.startswith("ddn/")})


def _oracle_inst(tag):
    from oracle import oracle as O
    if tag == "cfg1_v0.3":
        from b200_helpers import oracle_instance  # noqa: F401  (GPU helpers import the package)
    A = G.arrays()
    if tag.startswith("cfg1"):
        f = G.flat_inputs(tag)
    else:
        f = G.flat_inputs(f"small/{tag}")
    return O.build_instance(f["capacity"], f["demand0"], f["com_path_ptr0"], f["path_edge_ptr0"],
                            f["path_edges0"]), A


@pytest.mark.parametrize("tag", TAGS)
def test_oracle_reductions_vs_reference(tag):
    from oracle import oracle as O
    I, _ = _oracle_inst(tag)
    M = misc()
    for t in range(3):
        key = f"{tag}/t{t}"
        x, pv = M[f"{key}/x"], M[f"{key}/pv"]
        assert np.array_equal(O.commodity_sums(I, x), M[f"{key}/commodity_sums"]), key
        assert np.array_equal(O.edge_loads(I, x), M[f"{key}/edge_loads"]), key
        assert np.array_equal(O.edge_loads_from_pairs(I, pv), M[f"{key}/edge_loads_from_pairs"]), key
        for a in (0, 1, 2):
            got, want = O.score_paths(I, x, a), M[f"{key}/score_a{a}"]
            if a == 2:  # numpy's SIMD power in the reference vs glibc pow
                np.testing.assert_allclose(got, want, rtol=1e-15, atol=0)
            else:
                assert np.array_equal(got, want), (key, a)


def test_oracle_det_diff_norm_vs_reference():
    from oracle import oracle as O
    M = misc()
    for n in _lengths():
        assert O.det_diff_norm(M[f"ddn/{n}/a"], M[f"ddn/{n}/b"]) == M[f"ddn/{n}/out"][0], n


# ------------------------------------------------------------------ GPU


def _gpu_inst(tag):
    from b200_helpers import SMALL_BUILDERS, golden_instance
    return golden_instance(tag) if tag.startswith("cfg1") else SMALL_BUILDERS[tag]()


@pytest.mark.gpu
@pytest.mark.parametrize("tag", TAGS)
def test_gpu_reductions_vs_reference(tag):
    pf = pytest.importorskip("paper_2605_01748_b200")
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    inst = _gpu_inst(tag)
    M = misc()
    for t in range(3):
        key = f"{tag}/t{t}"
        x, pv = M[f"{key}/x"], M[f"{key}/pv"]
        assert np.array_equal(pf.commodity_sums(inst, x), M[f"{key}/commodity_sums"]), key
        assert np.array_equal(pf.edge_loads(inst, x), M[f"{key}/edge_loads"]), key
        assert np.array_equal(pf.edge_loads_from_pairs(inst, pv), M[f"{key}/edge_loads_from_pairs"]), key
        for a in (0, 1, 2):
            got, want = pf.score_paths(inst, x, a), M[f"{key}/score_a{a}"]
            if a == 2:  # CUDA pow vs numpy's SIMD power (both within 1 ulp of exact)
                np.testing.assert_allclose(got, want, rtol=1e-15, atol=0)
            else:
                assert np.array_equal(got, want), (key, a)


@pytest.mark.gpu
def test_gpu_det_diff_norm_vs_reference():
    pf = pytest.importorskip("paper_2605_01748_b200")
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    M = misc()
    for n in _lengths():
        assert pf.det_diff_norm(M[f"ddn/{n}/a"], M[f"ddn/{n}/b"]) == M[f"ddn/{n}/out"][0], n


@pytest.mark.gpu
def test_gpu_reductions_reject_wrong_lengths():
    """A short buffer is an InputError, not an out-of-bounds host read (the
    reference raises IndexError from the gather in the same case)."""
    pf = pytest.importorskip("paper_2605_01748_b200")
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    inst = _gpu_inst("chain")
    short = np.zeros(inst.num_paths - 1)
    for fn in (pf.commodity_sums, pf.edge_loads):
        with pytest.raises(pf.InputError):
            fn(inst, short)
    with pytest.raises(pf.InputError):
        pf.edge_loads_from_pairs(inst, np.zeros(inst.num_pairs + 1))
    with pytest.raises(pf.InputError):
        pf.score_paths(inst, short, 1)
    with pytest.raises(pf.InputError):
        pf.project(inst, short, 1)
