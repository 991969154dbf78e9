"""GPU: the batch-aware runner (harness.py) equals the reference's per-query
protocol (harness._Runner.query, harness.py:258-270) query for query, for every estimator."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_2107_02736_b200 as g  # noqa: E402
from oracle import deann_oracle as O  # noqa: E402
from paper_2107_02736_b200.harness import BatchRunner, evaluate_batch, relative_error  # noqa: E402


@pytest.fixture(scope="module")
def problem():
    rng = np.random.default_rng(61)
    centers = rng.normal(scale=3.0, size=(6, 8))
    X = (centers[rng.integers(0, 6, 3000)] + rng.normal(size=(3000, 8))).astype(np.float32)
    Q = centers[rng.integers(0, 6, 25)] + rng.normal(size=(25, 8))
    return X, Q, g.Dataset.from_array(X)


@pytest.mark.parametrize("estimator,params", [
    ("naive", {}), ("rs", {"m": 200}), ("rsp", {"m": 150}), ("deann", {"k": 20, "m": 100}),
    ("deannp", {"k": 20, "m": 100}), ("deann", {"k": 15, "m": 80, "n_clusters": 16, "n_probe": 3}),
])
def test_query_batch_equals_per_query_loop(problem, estimator, params):
    X, Q, ds = problem
    spec = g.KernelSpec("gaussian", 1.7)
    r1 = BatchRunner(estimator, ds, spec, params, seed=3)
    r2 = BatchRunner(estimator, ds, spec, params, seed=3)
    r1.reset(11)
    r2.reset(11)
    loop = [r1.query(y) for y in Q]
    batch = r2.query_batch(Q)
    assert len(batch) == len(loop)
    for a, b in zip(loop, batch):
        assert b.value == pytest.approx(a.value, rel=1e-12, abs=1e-300)
        assert (a.kernel_evals, a.neighbors_used, a.samples_used) == (b.kernel_evals, b.neighbors_used, b.samples_used)


def test_evaluate_batch_rows(problem):
    X, Q, ds = problem
    spec = g.KernelSpec("gaussian", 1.7)
    exact = O.naive_kde(O.Data(X), "gaussian", 1.7, Q)
    row, per_query = evaluate_batch("naive", ds, spec, Q, exact, {}, repetitions=2)
    assert row["mean_rel_err"] < 1e-5 and row["repetitions"] == 2 and len(per_query) == 2 * len(Q)
    row, _ = evaluate_batch("deann", ds, spec, Q, exact, {"k": 10, "m": 300, "n_clusters": 16, "n_probe": 16},
                            repetitions=3)
    assert row["recall"] == 1.0  # full probe = brute force (acceptance 7)
    assert 0 < row["mean_rel_err"] < 0.5 and row["mean_query_time_ms"] > 0
    rep = relative_error([1.0, 2.0, 5.0], [1.0, 4.0, 1e-20])
    assert rep.excluded_count == 1 and rep.mean_rel_err == pytest.approx(0.25)
