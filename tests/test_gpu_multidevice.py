"""Multi-device contexts (lt_create_devices / lt_create_mask) on
the one-GPU box: a group of members that share cuda:0 runs the whole
sharding path -- cost-balanced LPT partition, one host thread per member,
the gather of the sweeps' placement + frontier rows to the first member (peer
copies; NCCL needs distinct GPUs) and the scatter back to batch order -- and
must return exactly what the single-device context returns, statuses and
reference messages included. The single-device results are themselves
parity-tested against the compiled reference elsewhere."""
import numpy as np
import pytest

import paper_2508_08343_b200 as lt
from paper_2508_08343_b200 import _abi as A
from paper_2508_08343_b200.batch import ConditionBatch
from tests import workloads as W

pytestmark = pytest.mark.gpu

# per-run measurements, not results
VOLATILE = {"device_cycles", "phase_cycles"}


@pytest.fixture(scope="module")
def group3():
    g = lt.device_group([0, 0, 0])
    yield g
    g.close()


def same_summaries(a, b):
    assert len(a) == len(b)
    for name in a.dtype.names:
        if name in VOLATILE:
            continue
        assert np.array_equal(a[name], b[name], equal_nan=True), name


def test_group_shape(group3):
    assert group3.device_count() == 3
    assert group3.gather_transport() == "peer"  # repeated device: no NCCL communicator
    one = lt.device_group([0])
    try:
        assert one.device_count() == 1 and one.gather_transport() == "none"
    finally:
        one.close()


def test_group_simulate_matches_single(dev, group3):
    batch = W.c2_batch(duration_s=120.0, stride=5)
    cfg = lt.h100_like_config(32)
    a, _ = dev.simulate_batch(batch, cfg, want_digest=True)
    b, _ = group3.simulate_batch(batch, cfg, want_digest=True)
    same_summaries(a, b)
    t = group3.timing()
    assert t["devices"] == 3


def test_group_simulate_states_and_errors_match_single(dev, group3):
    batch, cfg = W.summary_cases()
    a, sa = dev.simulate_batch(batch, cfg, want_states=True, want_digest=True)
    na = [dev.message(i) for i in range(len(a))]
    b, sb = group3.simulate_batch(batch, cfg, want_states=True, want_digest=True)
    nb = [group3.message(i) for i in range(len(b))]
    same_summaries(a, b)
    assert na == nb
    for k in sa:
        assert np.array_equal(sa[k], sb[k], equal_nan=True), k


def test_group_sweep_matches_single(dev, group3):
    conds = W.c4_conditions()
    grid, opts, dur, seed = W.c4_grid()
    sel = [conds[i] for i in W.c4_sample_indices()[:24]]
    cb = ConditionBatch.from_conditions(sel)
    cfg = lt.h100_like_config(1)
    pa, fa = dev.sweep_batch(cb, cfg, grid, dur, seed, opts)
    pb, fb = group3.sweep_batch(cb, cfg, grid, dur, seed, opts)
    for name in pa.dtype.names:
        assert np.array_equal(pa[name], pb[name]), name
    assert np.array_equal(fa, fb)
    t = group3.timing()
    assert t["devices"] == 3 and t["gather_bytes"] > 0


def test_group_sweep_errors_keep_lowest_index(dev, group3):
    """A condition failing validation and one failing in the engine keep
    their indices and messages through the shard / gather / scatter."""
    conds, cfg, grid, dur, seed, opts = W.sweep_cases()
    conds = list(conds[:10])
    conds[6] = lt.Condition(mix=[], lengths=conds[6].lengths)  # ValidationError
    big = lt.Condition(mix=[lt.AdapterTemplate(rank=64, rate=0.5)], lengths=conds[3].lengths)
    conds[3] = big  # rank without a slot cost in a small config -> ConfigError per point
    cb = ConditionBatch.from_conditions(conds)
    pa, fa = dev.sweep_batch(cb, cfg, grid, dur, seed, opts)
    ma = [dev.message(i) for i in range(len(conds))]
    pb, fb = group3.sweep_batch(cb, cfg, grid, dur, seed, opts)
    mb = [group3.message(i) for i in range(len(conds))]
    for name in pa.dtype.names:
        assert np.array_equal(pa[name], pb[name]), name
    assert np.array_equal(fa, fb)
    assert ma == mb
    assert int(pa["status"][6]) == A.LT_ERR_VALIDATION


def test_group_dataset_matches_single(dev, group3, tmp_path):
    spec = lt.DatasetSpec(rates=[3.2, 0.4, 0.05], ranks=[8, 16], triple_size=2,
                          lengths=lt.LengthSpec.mean(250, 50, 231, 50), duration_s=60.0, seed=3,
                          grid=lt.SweepGrid(n_values=[1, 2, 4, 8, 16], g_mode=lt.GMode.Geometric),
                          sweep=lt.SweepOptions(early_exit=True, early_exit_k=2))
    cfg = lt.h100_like_config(1)
    a = tmp_path / "a.csv"
    b = tmp_path / "b.csv"
    pa = lt.api.run_generate_dataset(dev.lib, dev.ctx, spec, cfg, str(a))
    pb = lt.api.run_generate_dataset(group3.lib, group3.ctx, spec, cfg, str(b))
    assert a.read_bytes() == b.read_bytes()
    assert (pa.completed, pa.failed) == (pb.completed, pb.failed)
