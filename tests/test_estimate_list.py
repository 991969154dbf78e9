"""CPU: EstimateList (deann_batch's lazily built list[Estimate]) behaves as a list everywhere a
caller of the reference's deann_batch (estimators.py:382-410) would use one."""

import copy
import pickle

import numpy as np

from paper_2107_02736_b200.estimators import Estimate, EstimateList


def _mk(vals=(0.5, 0.25, 0.125)):
    return EstimateList(np.array(vals), 1100, 100, 1000)


def test_lazy_until_read_then_a_plain_list():
    L = _mk()
    assert isinstance(L, list) and len(L) == 3 and L._lazy
    assert np.array_equal(L.values, [0.5, 0.25, 0.125])  # arrays without materialising
    assert L._lazy
    assert L[1] == Estimate(0.25, 1100, 100, 1000)
    assert not L._lazy and list.__len__(L) == 3


def test_list_protocols():
    ref = [Estimate(v, 1100, 100, 1000) for v in (0.5, 0.25, 0.125)]
    assert _mk() == ref and list(_mk()) == ref and tuple(_mk()) == tuple(ref)
    assert [e.value for e in _mk()] == [0.5, 0.25, 0.125]
    assert sorted(_mk(), key=lambda e: e.value)[0].value == 0.125
    assert _mk()[-1].value == 0.125 and _mk()[1:] == ref[1:]
    assert ref[0] in _mk() and _mk().index(ref[2]) == 2 and _mk().count(ref[0]) == 1
    assert list(reversed(_mk())) == ref[::-1]
    assert _mk() + [1] == ref + [1] and [1] + _mk() == [1] + ref and _mk() * 2 == ref * 2
    L = _mk()
    L.append(ref[0])
    assert len(L) == 4
    L = _mk()
    L.sort(key=lambda e: e.value)
    assert L[0].value == 0.125
    assert bool(_mk()) and not bool(EstimateList(np.array([]), 0, 0, 0))
    assert repr(_mk()) == repr(ref)
    assert pickle.loads(pickle.dumps(_mk())) == ref and copy.deepcopy(_mk()) == ref and copy.copy(_mk()) == ref
    assert np.asarray(_mk()).shape == (3,)


def test_counters_and_flags():
    L = EstimateList(np.array([0.1, 0.2]), np.array([7, 9]), np.array([3, 5]), 4, truncated=np.array([True, False]),
                     clamped=False)
    assert [(e.kernel_evals, e.neighbors_used, e.samples_used, e.truncated, e.clamped) for e in L] == \
        [(7, 3, 4, True, False), (9, 5, 4, False, False)]
