"""Host-side logic of the drop-in API (no GPU): types, validation, grids,
half-grid index math, tolerance policy, error taxonomy, budgets, and the
loud failure when no CUDA device exists.  Mirrors pkg/tests/test_kernels.py.
"""

import numpy as np
import pytest

import paper_2506_05617_b200 as cs
from paper_2506_05617_b200 import configs, engine
from paper_2506_05617_b200.errors import NonFiniteWeight, ZeroDimension


def test_offsets_3x3_centered():
    offs = cs.neighborhood_offsets(3, 3)
    assert offs.shape == (9, 2)
    assert set(map(tuple, offs)) == {(a, b) for a in (-1, 0, 1) for b in (-1, 0, 1)}
    assert tuple(offs[4]) == (0, 0)


def test_offsets_even_extent_biased_negative():
    offs = cs.neighborhood_offsets(4, 3)
    assert sorted(set(offs[:, 0])) == [-2, -1, 0, 1]
    assert sorted(set(offs[:, 1])) == [-1, 0, 1]
    assert offs.tolist()[:4] == [[-2, -1], [-2, 0], [-2, 1], [-1, -1]]


@pytest.mark.parametrize("kh,kw", [(1, 1), (2, 5), (3, 3), (4, 4), (5, 2)])
def test_offsets_match_oracle(orc, kh, kw):
    assert np.array_equal(cs.neighborhood_offsets(kh, kw), orc.offsets(kh, kw))


def test_offsets_reject_zero_extent():
    with pytest.raises(ZeroDimension):
        cs.neighborhood_offsets(0, 3)


def test_validate_reports_nan_index():
    w = np.zeros((1, 1, 3, 3))
    w[0, 0, 1, 1] = np.nan
    with pytest.raises(NonFiniteWeight) as err:
        cs.validate_kernel(cs.ConvKernel(weights=w))
    assert err.value.index == (0, 0, 1, 1)


def test_validate_zero_channel_and_precision():
    with pytest.raises(ZeroDimension):
        cs.validate_kernel(cs.ConvKernel(weights=np.zeros((0, 1, 3, 3))))
    with pytest.raises(ZeroDimension):
        cs.validate_kernel(cs.ConvKernel(weights=np.zeros((1, 1, 3, 3)), precision="f16"))


def test_from_array_precision_tag():
    assert cs.ConvKernel.from_array(np.zeros((1, 1, 1, 1), np.float32)).precision == "f32"
    k = cs.ConvKernel.from_array(np.zeros((1, 1, 1, 1)))
    assert k.precision == "f64" and k.weights.dtype == np.float64


def test_taps_layout(orc):
    k = cs.random_kernel(3, 2, 3, 4, seed=5)
    assert np.array_equal(k.taps(), orc.taps(k.weights))


def test_grid_ordering_and_negation():
    grid = cs.FrequencyGrid(cs.SpatialDims(n=2, m=3))
    assert np.allclose(grid.frequencies, [(i / 2, j / 3) for i in range(2) for j in range(3)])
    assert grid.index_of(1, 2) == 5
    g = cs.FrequencyGrid(cs.SpatialDims(n=4, m=6))
    pts = {tuple(np.round(k, 12)) for k in g.frequencies}
    assert {tuple(np.round((-np.asarray(k)) % 1.0, 12)) for k in pts} == pts


def test_random_kernel_deterministic_and_dists():
    a = cs.random_kernel(2, 3, 3, 3, seed=9)
    assert np.array_equal(a.weights, cs.random_kernel(2, 3, 3, 3, seed=9).weights)
    assert not np.array_equal(a.weights, cs.random_kernel(2, 3, 3, 3, seed=10).weights)
    u = cs.random_kernel(4, 4, 3, 3, seed=1, dist="uniform")
    assert (u.weights >= -1).all() and (u.weights < 1).all()
    with pytest.raises(ValueError):
        cs.random_kernel(1, 1, 1, 1, dist="cauchy")


def test_spatial_dims_validation():
    with pytest.raises(ZeroDimension):
        cs.SpatialDims(n=0, m=4)


@pytest.mark.parametrize("n,m", [(1, 1), (1, 5), (2, 2), (2, 3), (3, 3), (4, 6), (5, 3), (7, 8),
                                 (56, 56), (256, 256), (7, 7), (28, 28), (64, 64)])
def test_half_grid_representatives(n, m):
    F = n * m
    f = np.arange(F)
    i, j = f // m, f % m
    fs = ((n - i) % n) * m + (m - j) % m
    brute = f[f <= fs]
    reps = engine.half_grid_indices(n, m)
    assert np.array_equal(reps, brute)
    s = engine.self_conjugate_count(n, m)
    assert engine.half_grid_count(n, m) == len(brute) == (F + s) // 2
    rep_of, conj = engine.partner_map(n, m)
    assert np.array_equal(reps[rep_of], np.where(conj, fs, f))
    assert (conj == (f > fs)).all()


def test_half_grid_count_matches_library():
    lib = pytest.importorskip("paper_2506_05617_b200._lib").load()
    for n, m in [(1, 1), (2, 3), (5, 3), (56, 56), (256, 256), (7, 8)]:
        assert lib.cs_half_grid_count(n, m) == engine.half_grid_count(n, m)


def test_effective_tol_policy():
    assert engine.effective_tol(1e-13, "f64", 256) == 1e-13
    assert engine.effective_tol(1e-13, "f32", 64) == pytest.approx(2.5e-6)
    assert engine.effective_tol(1e-13, "f32", 256) == pytest.approx(5e-6)
    assert engine.effective_tol(1e-3, "f32", 256) == 1e-3


def test_configs_match_baseline():
    w = configs.WORKLOADS
    assert [l.sv_count for l in w[1].layers] == [16 * 1024]
    assert w[2].sv_count == 64 * 4096 and w[2].vectors
    assert w[3].sv_count == 128 * 56 * 56 and not w[3].vectors
    assert len(w[4].layers) == 16 and w[4].sv_count == 1505280
    assert w[5].sv_count == 16777216 and w[5].vectors
    w1 = configs.layer_weights(w[1].layers[0])
    assert w1.dtype == np.float32 and w1.shape == (16, 16, 3, 3)
    assert abs(w1.std() - np.sqrt(2 / (16 * 9))) < 0.02


def test_sample_frequencies_include_self_conjugate():
    f = configs.sample_frequencies(256, 256, 32, seed=5)
    for sc in (0, 128, 128 * 256, 128 * 256 + 128):
        assert sc in f
    assert len(f) == 32 and np.all(np.diff(f) > 0)


def test_sort_descending_stable():
    assert cs.sort_descending(np.array([1.0, 3.0, 1.0, 2.0])).tolist() == [3.0, 2.0, 1.0, 1.0]


def test_phase_timings_reconcile():
    t = cs.PhaseTimings.build(0.5, 1.25, 0.25)
    assert t.s_total == t.s_transform + t.s_svd + t.s_copy


def test_budget_helpers(monkeypatch):
    assert cs.mem_budget_bytes(1.0) == 2**30
    monkeypatch.setenv("CONV_SPECTRA_MEM_BUDGET_GIB", "0.5")
    assert cs.mem_budget_bytes() == 2**29
    with pytest.raises(cs.AllocationFailure):
        engine.check_budget(10, 5, "x")


def test_method_and_boundary_validation():
    k = cs.random_kernel(1, 1, 1, 1)
    d = cs.SpatialDims(2, 2)
    with pytest.raises(ValueError):
        cs.compute_spectrum(k, d, method="svd")
    with pytest.raises(ValueError):
        cs.compute_spectrum(k, d, boundary="neumann")
    with pytest.raises(ValueError):
        cs.compute_spectrum(k, d, boundary="dirichlet")
    with pytest.raises(NotImplementedError):
        cs.compute_spectrum(k, d, method="explicit")


def test_no_cpu_fallback_without_cuda():
    import torch

    if torch.cuda.is_available():
        pytest.skip("CUDA present: the loud-failure path is only reachable without a GPU")
    with pytest.raises(RuntimeError, match="CUDA"):
        cs.compute_spectrum(cs.random_kernel(2, 2, 3, 3), cs.SpatialDims(4, 4))
    with pytest.raises(RuntimeError, match="CUDA"):
        cs.build_symbol_field(cs.random_kernel(2, 2, 3, 3), cs.SpatialDims(4, 4))


def test_materialize_on_host_triplet():
    # the global vector layout of blocksvd.py:306-311 on a synthetic triplet
    t = cs.SvdTriplet(k=(0.0, 0.0), U=np.eye(2, dtype=complex), sigma=np.ones(2),
                      V=np.eye(2, dtype=complex))
    v = cs.materialize_singular_vector(t, 0, "left", cs.SpatialDims(4, 4))
    assert v.shape == (32,)
    nz = v[np.abs(v) > 1e-14]
    assert len(nz) == 16 and np.allclose(np.abs(nz), 0.25)
    with pytest.raises(cs.IndexOutOfRange):
        cs.materialize_singular_vector(t, 2, "left", cs.SpatialDims(4, 4))
    with pytest.raises(ValueError):
        cs.materialize_singular_vector(t, 0, "up", cs.SpatialDims(4, 4))


@pytest.mark.parametrize("depth", [3, 8])
@pytest.mark.parametrize("n,m,u0,count", [(256, 256, 0, None), (64, 64, 100, 900), (7, 6, 0, None)])
def test_warm_plan_is_a_bfs_forest(depth, n, m, u0, count):
    """engine.warm_plan: every representative of the range solved exactly
    once; stage 0 cold seeds, every later block warm-started from a lattice
    neighbour (|di| + |dj| == 1) solved in the previous stage."""
    total = engine.half_grid_count(n, m)
    count = total - u0 if count is None else count
    plan = engine.warm_plan(n, m, u0, count, "cpu", depth)
    reps = engine.half_grid_indices(n, m)[u0:u0 + count]
    stage_of = np.full(count, -1)
    for d, (ids, pred) in enumerate(plan):
        ids = ids.numpy()
        assert (stage_of[ids] == -1).all()
        stage_of[ids] = d
        if d == 0:
            assert pred is None
            continue
        pred = pred.numpy()
        assert (stage_of[pred] >= 0).all() and (stage_of[pred] < d).all()
        di = np.abs(reps[ids] // m - reps[pred] // m)
        dj = np.abs(reps[ids] % m - reps[pred] % m)
        assert ((di + dj) == 1).all()
    assert (stage_of >= 0).all()
