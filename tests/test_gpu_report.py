"""Full simulation report on the device (lt_simulate_report):
the IterationTraceRow trace (engine.cpp:137-140), the LoadEvent list (:141)
and every request's token_emit_times_s (:132) -- the inputs of the
reference's simulation_report_json (json_io.cpp:608-687) -- bit-exact against
the compiled reference's own SimulationResult, and against the hand-traced
fixture's timeline (proj/tests/fixtures/hand_traced_two_adapter.json)."""
import json
import os

import numpy as np
import pytest

import paper_2508_08343_b200 as lt
from paper_2508_08343_b200 import _abi as A
from paper_2508_08343_b200.batch import WorkloadBatch, sim_options
from tests import workloads as W
from tests.conftest import GOLDEN

pytestmark = pytest.mark.gpu

VOLATILE = {"device_cycles", "phase_cycles", "sum_running", "sum_visited", "sum_arrivals", "sum_moves", "digest"}


def assert_reports_equal(dev, ref, batch, cfg, where=""):
    opts = sim_options(None, False, -1, False, report=True)
    g, gs, gr = dev.runner.report(batch, cfg, opts)
    r, rs, rr = ref.report(batch, cfg, opts)
    for f in ("status", "iterations", "load_events", "tokens_total", "preemptions", "final_clock_s",
              "throughput_tok_s", "ttft_mean_s", "itl_mean_s"):  # the report path's ITL mean is exact
        np.testing.assert_array_equal(g[f], r[f], err_msg=where + f)
    for k in gs:
        np.testing.assert_array_equal(gs[k], rs[k], err_msg=where + k)
    ok = g["status"] == A.LT_OK
    for i in np.nonzero(ok)[0]:
        n_it = int(g["iterations"][i])
        a = gr["trace"][gr["trace_offset"][i]:gr["trace_offset"][i] + n_it]
        b = rr["trace"][rr["trace_offset"][i]:rr["trace_offset"][i] + n_it]
        np.testing.assert_array_equal(a, b, err_msg=f"{where}trace of scenario {i}")
        n_ld = int(g["load_events"][i])
        a = gr["loads"][gr["load_offset"][i]:gr["load_offset"][i] + n_ld]
        b = rr["loads"][rr["load_offset"][i]:rr["load_offset"][i] + n_ld]
        np.testing.assert_array_equal(a, b, err_msg=f"{where}loads of scenario {i}")
        r0 = int(gs["req_offset"][i])
        for j in range(r0, r0 + int(g["n_requests"][i])):
            t = int(gs["tokens_generated"][j])
            a = gr["emit_times"][gr["emit_offset"][j]:gr["emit_offset"][j] + t]
            b = rr["emit_times"][rr["emit_offset"][j]:rr["emit_offset"][j] + t]
            np.testing.assert_array_equal(a, b, err_msg=f"{where}emit times of request row {j}")
    return g, gs, gr


def test_report_hand_traced_fixture(dev):
    fx = json.load(open(os.path.join(GOLDEN, "hand_traced_two_adapter.json")))
    cfg = W.fixture_config(fx)
    ads, reqs = W.fixture_scripted(fx)
    res = lt.run_scripted(reqs, ads, fx["duration_s"], cfg, dev=dev,
                          options=lt.SimOptions(record_iteration_trace=True))
    exp = fx["expected"]
    tol = fx["tolerance"]
    assert len(res.iteration_trace) == exp["iterations"]
    assert [t.iteration for t in res.iteration_trace] == list(range(exp["iterations"]))
    assert len(res.load_event_list) == len(exp["load_events"])
    for e, x in zip(res.load_event_list, exp["load_events"]):
        assert abs(e.time_s - x["time_s"]) <= tol and e.adapter_id == x["adapter_id"] and e.rank == x["rank"]
        assert e.source == lt.LoadSource.Cpu and abs(e.latency_s - x["latency_s"]) <= tol
    for r, x in zip(res.requests, exp["requests"]):
        assert len(r.token_emit_times_s) == len(x["emit_times_s"])
        for t, u in zip(r.token_emit_times_s, x["emit_times_s"]):
            assert abs(t - u) <= tol


def test_report_summary_cases_match_reference(dev, ref):
    batch, cfg = W.summary_cases()
    assert_reports_equal(dev, ref, batch, cfg)


@pytest.mark.parametrize("block", range(2))
def test_report_scripted_fuzz_match_reference(dev, ref, block):
    """Preemption-heavy scripted engines: stints split by preemptions and
    re-admissions, sole-survivor failures (no report rows), slot churn."""
    pre = 0
    for seed in range(block * 40, block * 40 + 40):
        ads, reqs, cfg = W.scripted_fuzz(seed, n_requests=40 + seed % 50, n_adapters=1 + seed % 6,
                                         tight=seed % 5 != 4)
        b = WorkloadBatch.from_workloads([W.scripted_workload(ads, 6.0)], scripted=[reqs])
        g, _, _ = assert_reports_equal(dev, ref, b, cfg, where=f"seed {seed}: ")
        pre += int(g["preemptions"].sum())
    assert pre > 0


def test_report_c2_subset_match_reference(dev, ref):
    batch = W.c2_batch(duration_s=120.0, stride=37)
    assert_reports_equal(dev, ref, batch, lt.h100_like_config(32))


def test_run_simulation_returns_full_result(dev, ref):
    wl = lt.WorkloadSpec(adapters=[lt.AdapterSpec(k + 1, (8, 16, 32)[k % 3], 0.3) for k in range(12)],
                         lengths=lt.LengthSpec.mean(250, 50, 231, 50), duration_s=120.0, seed=11)
    cfg = lt.h100_like_config(4)
    res = lt.run_simulation(wl, cfg, dev=dev, options=lt.SimOptions(record_iteration_trace=True))
    assert len(res.iteration_trace) == res.iterations
    assert len(res.load_event_list) == res.load_events
    for r in res.requests:
        assert len(r.token_emit_times_s) == r.tokens_generated
        if r.tokens_generated:
            assert r.token_emit_times_s[0] == r.first_token_time_s
            assert all(np.diff(r.token_emit_times_s) > 0)
    last = max((r.token_emit_times_s[-1] for r in res.requests if r.tokens_generated), default=0.0)
    assert last == res.final_clock_s
    # throughput = emits inside the window / duration (metrics.cpp:96)
    emits = sum(sum(1 for t in r.token_emit_times_s if t <= wl.duration_s) for r in res.requests)
    assert res.metrics.throughput_tok_s == emits / wl.duration_s


def test_reference_side_binding_prints_identical_reports():
    """The reference's own code through integration/gpu_backend.cpp: its
    simulation_report_json / placement_result_to_json print byte-identical
    documents for the GPU results and for its own run_simulation /
    run_scripted / sweep_optimal (oracle/_ref/gpu_backend_check, built with
    the oracle where /root/reference exists)."""
    import subprocess

    from oracle import pyoracle

    if not os.path.exists(pyoracle.SHIM_CHECK):
        pytest.skip("oracle/_ref/gpu_backend_check not built (needs /root/reference at build time)")
    p = subprocess.run([pyoracle.SHIM_CHECK], capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stdout[-4000:] + p.stderr[-2000:]
    assert p.stdout.startswith("ok: ")
