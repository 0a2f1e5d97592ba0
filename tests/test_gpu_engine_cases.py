"""The reference's own engine tests (proj/tests/test_engine.cpp), run on the
B200 path through the mirrored API with the same inputs and expectations.
Per-token emit vectors are not materialised on the device; where the
reference checks them, the first/last emit (first_token_time_s /
completion_time_s), token counts and iteration counts pin the same timeline,
and the whole run is also diffed against the compiled reference.
"""
import math

import numpy as np
import pytest

import paper_2508_08343_b200 as lt
from paper_2508_08343_b200.batch import WorkloadBatch, sim_options
from tests import workloads as W

pytestmark = pytest.mark.gpu

Phase = lt.Phase


def tiny_config(kv_budget, k5=0.1):
    """test_engine.cpp:87-97: single slot, step = k5, +0.5 s per rank-8 load."""
    return lt.ServerConfig(slots=1, latency=lt.LatencyCoefficients(k5=k5, k7=1.0),
                           memory=lt.MemoryModel(total_kv_budget=kv_budget, slot_cost_table={8: 100}),
                           load=lt.LoadLatencyTable(cpu_load_seconds={8: 0.5}))


def base_model_config():
    return lt.ServerConfig(slots=1, latency=lt.LatencyCoefficients(k5=0.05),
                           memory=lt.MemoryModel(total_kv_budget=1000, slot_cost_base_rank8=10.0))


def req(i, a, t, n_in, n_out):
    return lt.Request(i, a, t, n_in, n_out)


def close(x, y):
    return math.isclose(x, y, rel_tol=1e-12, abs_tol=0.0)


def same_as_reference(dev, ref, reqs, ads, duration, cfg, opts=None):
    b = WorkloadBatch.from_workloads([W.scripted_workload(ads, duration)], scripted=[reqs])
    g, gs = dev.simulate_batch(b, cfg, options=opts, want_states=True, want_digest=True)
    r, rs = ref.simulate(b, cfg, sim_options(opts, True), want_states=True)
    for f in ("status", "iterations", "digest", "final_clock_s", "load_events", "preemptions", "truncated"):
        assert g[0][f] == r[0][f], f
    for k in gs:
        np.testing.assert_array_equal(gs[k], rs[k], err_msg=k)


def test_base_model_traffic(dev, ref):  # test_engine.cpp:165-189
    ads, reqs = [lt.AdapterSpec(7, 0, 0.0)], [req(0, 7, 0.0, 1, 3)]
    res = lt.run_scripted(reqs, ads, 1.0, base_model_config(), lt.SimOptions(check_invariants=True), dev=dev)
    assert res.iterations == 3
    assert res.load_events == 0
    assert res.kv_capacity_tokens == 1000
    r = res.requests[0]
    assert r.tokens_generated == 3
    assert close(r.first_token_time_s, 0.05) and close(r.completion_time_s, 0.15)
    assert close(res.final_clock_s, 0.15)
    same_as_reference(dev, ref, reqs, ads, 1.0, base_model_config())


def test_kv_pressure_preempts_younger(dev, ref):  # test_engine.cpp:191-221
    cfg = tiny_config(116)
    ads, reqs = [lt.AdapterSpec(1, 8, 0.0)], [req(0, 1, 0.0, 5, 5), req(1, 1, 0.0, 5, 5)]
    res = lt.run_scripted(reqs, ads, 1.0, cfg, lt.SimOptions(check_invariants=True), dev=dev)
    r0, r1 = res.requests
    assert r0.phase == Phase.Finished and r1.phase == Phase.Finished
    assert r0.preemption_count == 0 and r1.preemption_count == 1
    assert r0.tokens_generated == 5 and r1.tokens_generated == 5
    # emits r0 {0.6, 0.7, 0.8, 0.9, 1.0}, r1 {0.6, 0.7, 0.8, 1.1, 1.2}
    assert close(r0.first_token_time_s, 0.6) and close(r0.completion_time_s, 1.0)
    assert close(r1.first_token_time_s, 0.6) and close(r1.completion_time_s, 1.2)
    assert res.load_events == 1
    assert res.iterations == 7
    same_as_reference(dev, ref, reqs, ads, 1.0, cfg)


def test_never_fitting_request_is_rejected(dev, ref):  # test_engine.cpp:223-234
    cfg = tiny_config(116)
    ads, reqs = [lt.AdapterSpec(1, 8, 0.0)], [req(0, 1, 0.0, 20, 2), req(1, 1, 0.0, 5, 2)]
    res = lt.run_scripted(reqs, ads, 1.0, cfg, dev=dev)
    assert res.requests[0].phase == Phase.Rejected and res.requests[0].tokens_generated == 0
    assert res.requests[1].phase == Phase.Finished and res.requests[1].tokens_generated == 2
    same_as_reference(dev, ref, reqs, ads, 1.0, cfg)


def test_sole_survivor(dev, ref):  # test_engine.cpp:236-251
    cfg = tiny_config(107)
    ads = [lt.AdapterSpec(1, 8, 0.0)]
    with pytest.raises(lt.SimulationError, match="single request exceeds KV capacity"):
        lt.run_scripted([req(0, 1, 0.0, 5, 4)], ads, 1.0, cfg, dev=dev)
    res = lt.run_scripted([req(0, 1, 0.0, 5, 3)], ads, 1.0, cfg, lt.SimOptions(check_invariants=True), dev=dev)
    assert res.requests[0].phase == Phase.Finished and res.requests[0].tokens_generated == 3
    same_as_reference(dev, ref, [req(0, 1, 0.0, 5, 3)], ads, 1.0, cfg)


def test_iteration_cap_truncates(dev, ref):  # test_engine.cpp:253-265
    cfg = tiny_config(1000)
    ads, reqs = [lt.AdapterSpec(1, 8, 0.0)], [req(0, 1, 0.0, 5, 50)]
    opts = lt.SimOptions(iteration_cap_override=2)
    res = lt.run_scripted(reqs, ads, 1.0, cfg, opts, dev=dev)
    assert res.truncated and res.iterations == 2
    assert res.requests[0].tokens_generated == 2 and res.requests[0].phase == Phase.Running
    same_as_reference(dev, ref, reqs, ads, 1.0, cfg, opts)


def test_empty_script_drains(dev):  # test_engine.cpp:267-275
    res = lt.run_scripted([], [lt.AdapterSpec(1, 8, 0.0)], 1.0, tiny_config(1000), dev=dev)
    assert res.iterations == 0 and res.requests == [] and res.final_clock_s == 0.0 and not res.truncated


def test_idle_jump(dev, ref):  # test_engine.cpp:277-295
    ads, reqs = [lt.AdapterSpec(7, 0, 0.0)], [req(0, 7, 0.0, 1, 2), req(1, 7, 100.0, 1, 2)]
    res = lt.run_scripted(reqs, ads, 101.0, base_model_config(), dev=dev)
    assert res.iterations == 4
    r1 = res.requests[1]
    assert close(r1.first_token_time_s, 100.05) and close(r1.completion_time_s, 100.10)
    assert close(res.final_clock_s, 100.10)
    same_as_reference(dev, ref, reqs, ads, 101.0, base_model_config())


def test_scripted_validation(dev):  # test_engine.cpp:297-312
    cfg, ads = tiny_config(1000), [lt.AdapterSpec(1, 8, 0.0)]
    with pytest.raises(lt.ValidationError):
        lt.run_scripted([req(5, 1, 0.0, 5, 2)], ads, 1.0, cfg, dev=dev)
    with pytest.raises(lt.ValidationError):
        lt.run_scripted([req(0, 9, 0.0, 5, 2)], ads, 1.0, cfg, dev=dev)
    with pytest.raises(lt.ValidationError):
        lt.run_scripted([], [], 1.0, cfg, dev=dev)
    with pytest.raises(lt.ValidationError):
        lt.run_scripted([], ads, 0.0, cfg, dev=dev)


def test_slots_eating_the_budget_are_rejected(dev):  # test_engine.cpp:314-319
    with pytest.raises(lt.ConfigError):
        lt.run_scripted([req(0, 1, 0.0, 5, 2)], [lt.AdapterSpec(1, 8, 0.0)], 1.0, tiny_config(100), dev=dev)


def test_seed_determinism(dev):  # test_engine.cpp:321-348
    wl = lt.WorkloadSpec(adapters=[lt.AdapterSpec(1, 8, 2.0), lt.AdapterSpec(2, 16, 1.0)],
                         lengths=lt.LengthSpec.mean(20.0, 5.0, 10.0, 3.0), duration_s=20.0, seed=42)
    cfg = lt.h100_like_config(2)
    a = lt.run_simulation(wl, cfg, dev=dev)
    b = lt.run_simulation(wl, cfg, dev=dev)
    assert len(a.requests) == len(b.requests) > 10
    assert (a.iterations, a.final_clock_s, a.load_events, a.digest) == (b.iterations, b.final_clock_s,
                                                                        b.load_events, b.digest)
    assert [(r.first_token_time_s, r.completion_time_s, r.preemption_count) for r in a.requests] == \
           [(r.first_token_time_s, r.completion_time_s, r.preemption_count) for r in b.requests]
    wl.seed = 43
    c = lt.run_simulation(wl, cfg, dev=dev)
    assert c.final_clock_s != a.final_clock_s


def test_step_latency_trace(dev, ref):  # test_engine.cpp:350-362 (trace rows: 0.6 s with the load, then 0.1 s)
    cfg = tiny_config(1000)
    ads, reqs = [lt.AdapterSpec(1, 8, 0.0)], [req(0, 1, 0.0, 5, 2)]
    res = lt.run_scripted(reqs, ads, 1.0, cfg, dev=dev)
    assert res.iterations == 2 and res.load_events == 1
    r = res.requests[0]
    assert close(r.first_token_time_s, 0.6) and close(r.completion_time_s - r.first_token_time_s, 0.1)
    same_as_reference(dev, ref, reqs, ads, 1.0, cfg)
