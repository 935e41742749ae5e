"""Host-side logic on CPU: synthetic generator, boundary types."""
import numpy as np
import pytest

from paper_1708_08640_b200 import api, synth


def test_distinct_coords_are_distinct_and_in_range():
    rng = np.random.Generator(np.random.PCG64(1))
    c = synth.distinct_coords(5000, [30, 40, 50], [("zipf", 1.2), "uniform", "uniform"], rng)
    assert c.shape == (5000, 3)
    assert np.unique(c, axis=0).shape[0] == 5000
    assert c.min() >= 0 and (c < np.array([30, 40, 50])).all()
    # Zipf mode is skewed towards index 0
    counts = np.bincount(c[:, 0], minlength=30)
    assert counts[0] > 3 * counts[10]


def test_planted_values_match_brute_force():
    rng = np.random.Generator(np.random.PCG64(2))
    core = rng.random((2, 3, 4))
    F = [rng.random((5, 2)), rng.random((6, 3)), rng.random((7, 4))]
    idx = np.array([[0, 1, 2], [4, 5, 6], [3, 0, 1]])
    got = synth.planted_values(core, F, idx)
    want = [np.einsum("abc,a,b,c->", core, F[0][i], F[1][j], F[2][k]) for i, j, k in idx]
    np.testing.assert_allclose(got, want, rtol=1e-12)


def test_generator_is_deterministic_and_shaped():
    spec = synth.config1(literal=False)
    spec.nnz, spec.dims = 3000, [40, 40, 40]
    spec.matrices[0].cols, spec.matrices[0].nnz = 20, 300
    b1, t1, _ = synth.generate(spec)
    b2, t2, _ = synth.generate(spec)
    np.testing.assert_array_equal(b1.tensor.indices, b2.tensor.indices)
    np.testing.assert_array_equal(b1.tensor.values, b2.tensor.values)
    assert b1.tensor.nnz == 2700 and t1.nnz == 300
    m = b1.matrices[0]
    assert m.rows == 40 and m.cols == 20 and m.nnz == 300


def test_symmetric_matrix_is_symmetric():
    spec = synth.config2(scale=1e-4)
    spec.dims = [500, 500, 50]
    spec.matrices[0].cols = 500
    b, _, _ = synth.generate(spec)
    m = b.matrices[0]
    pairs = {(int(i), int(j)): v for (i, j), v in zip(m.indices, m.values)}
    for (i, j), v in pairs.items():
        assert pairs[(j, i)] == v


def test_boundary_type_validation():
    with pytest.raises(api.ValidationError):
        api.SparseTensor([3, 3], [[0, 0], [1, 1]], [1.0])
    t = api.SparseTensor([3, 3, 3], [[0, 0, 0]], [1.0])
    with pytest.raises(api.ValidationError):
        api.make_bundle(t, [api.CoupledMatrix(0, 4, 2, [[0, 0]], [1.0])])
    with pytest.raises(api.ValidationError):
        api.make_bundle(t, [api.CoupledMatrix(3, 3, 2, [[0, 0]], [1.0])])
