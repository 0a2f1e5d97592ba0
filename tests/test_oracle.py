"""The oracle itself, checked on CPU (no GPU): the C restatement
(oracle/restate.c, `ltor_*`) must reproduce the reference's own golden
vectors (tests/golden, generated from the compiled reference and the
reference's JSON fixtures) and -- where oracle/_ref is built -- the compiled
reference bit for bit."""
import json
import math
import os
import struct

import numpy as np
import pytest

import paper_2508_08343_b200 as lt
from paper_2508_08343_b200.batch import ConditionBatch, WorkloadBatch, sim_options
from tests import workloads as W
from tests.conftest import GOLDEN

SKIP = ("device_cycles", "phase_cycles", "sum_visited", "sum_arrivals", "sum_moves", "_pad")


def unhex(h):
    return struct.unpack("<d", bytes.fromhex(h))[0]


def derived_values_case():
    """derived_values.json lat_step: R=10, W=5, g=4, n=8, a=1, one rank-8 load of 0.05 s."""
    dv = json.load(open(os.path.join(GOLDEN, "derived_values.json")))["lat_step"]
    x = dv["inputs"]
    cfg = lt.ServerConfig(slots=x["g"], latency=lt.LatencyCoefficients(x["k1"], x["k2"], x["k3"], x["k4"], x["k5"],
                                                                       x["k6"], x["k7"]),
                          memory=lt.MemoryModel(total_kv_budget=4 + 100, slot_cost_table={8: 1}),
                          load=lt.LoadLatencyTable(cpu_load_seconds={int(k): v for k, v in x["cpu_load_seconds"].items()}))
    ads = [lt.AdapterSpec(k + 1, 8, 1.0) for k in range(x["n"])]
    reqs = [lt.Request(i, 1, 0.0, 9, 5) for i in range(x["r_running"] + x["r_waiting"])]
    return cfg, ads, reqs, dv["expected_s"]


def test_hand_traced_fixture(port):
    fx = json.load(open(os.path.join(GOLDEN, "hand_traced_two_adapter.json")))
    cfg = W.fixture_config(fx)
    ads, reqs = W.fixture_scripted(fx)
    b = WorkloadBatch.from_workloads([W.scripted_workload(ads, fx["duration_s"])], scripted=[reqs])
    out, st = port.simulate(b, cfg, sim_options(), want_states=True)
    exp = fx["expected"]
    assert out[0]["iterations"] == exp["iterations"]
    assert abs(out[0]["final_clock_s"] - exp["final_clock_s"]) <= fx["tolerance"]
    assert out[0]["load_events"] == len(exp["load_events"])
    for i, e in enumerate(exp["requests"]):
        assert abs(st["first_token_time_s"][i] - st["arrival_time_s"][i] - e["ttft_s"]) <= fx["tolerance"]
        assert abs(st["completion_time_s"][i] - e["completion_s"]) <= fx["tolerance"]


def test_derived_lat_step(port):
    cfg, ads, reqs, want = derived_values_case()
    b = WorkloadBatch.from_workloads([W.scripted_workload(ads, 10.0)], scripted=[reqs])
    out, _ = port.simulate(b, cfg, sim_options(lt.SimOptions(iteration_cap_override=1)))
    assert out[0]["truncated"] == 1 and out[0]["iterations"] == 1
    assert math.isclose(out[0]["final_clock_s"], want, rel_tol=1e-12)


def test_arrivals_golden(port):
    gold = json.load(open(os.path.join(GOLDEN, "arrivals.json")))
    if gold["libm_variant"] != ("fma" if lt.load_library().host_libm_variant() else "generic"):
        pytest.skip("golden arrivals were generated under the other glibc libm build")
    reqs, counts = port.generate_arrivals(WorkloadBatch.from_workloads(W.arrival_cases()), sim_options())
    offs = np.concatenate([[0], np.cumsum(counts)])
    for c in gold["cases"]:
        rr = reqs[offs[c["case"]]:offs[c["case"] + 1]]
        assert len(rr) == c["n"]
        assert rr["adapter_id"].tolist() == c["adapter_id"]
        assert rr["input_tokens"].tolist() == c["input_tokens"]
        assert rr["output_tokens"].tolist() == c["output_tokens"]
        assert [struct.pack("<d", x).hex() for x in rr["arrival_time_s"]] == c["arrival_hex"]


def test_summaries_golden(port):
    gold = json.load(open(os.path.join(GOLDEN, "summaries.json")))["records"]
    b, cfg = W.summary_cases()
    out, _ = port.simulate(b, cfg, sim_options(None, True))
    for i, rec in enumerate(gold):
        for k, v in rec.items():
            if k in SKIP:
                continue
            got = out[i][k]
            if isinstance(v, str):
                assert got == unhex(v), (i, k)  # the restatement is bit-exact, ITL included
            else:
                assert int(got) == v, (i, k)


def test_sweeps_golden(port):
    gold = json.load(open(os.path.join(GOLDEN, "sweeps.json")))["records"]
    conds, cfg, grid, dur, seed, opts = W.sweep_cases()
    pl, fr = port.sweep(ConditionBatch.from_conditions(conds), cfg, grid, dur, seed, opts, sim_options())
    for i, rec in enumerate(gold):
        p = pl[i]
        assert int(p["status"]) == rec["status"]
        assert (int(p["n_star"]), int(p["g_star"]), int(p["all_starved"]), int(p["frontier_open"])) == \
            (rec["n_star"], rec["g_star"], rec["all_starved"], rec["frontier_open"])
        assert struct.pack("<d", p["max_throughput_tok_s"]).hex() == rec["max_throughput_hex"]
        got = [[int(f["n"]), int(f["g"]), struct.pack("<d", f["throughput_tok_s"]).hex(), int(f["starved"]),
                int(f["skipped"])] for f in fr[i][:int(p["frontier_count"])]]
        assert got == rec["frontier"]


@pytest.mark.parametrize("priority", [True, False])
def test_port_matches_reference_fuzz(port, ref, priority):
    for seed in range(60):
        ads, reqs, cfg = W.scripted_fuzz(seed + (0 if priority else 1000), n_requests=30 + seed % 60,
                                         n_adapters=1 + seed % 6, tight=seed % 5 != 4)
        cfg.loaded_adapter_priority = priority
        b = WorkloadBatch.from_workloads([W.scripted_workload(ads, 6.0)], scripted=[reqs])
        r, rs = ref.simulate(b, cfg, sim_options(None, True), want_states=True)
        p, ps = port.simulate(b, cfg, sim_options(None, True), want_states=True)
        for f in r.dtype.names:
            if f not in SKIP:
                assert np.array_equal(r[f], p[f]), (seed, f)
        assert ref.message(0) == port.message(0)
        if r[0]["status"] == 0:
            for k in rs:
                np.testing.assert_array_equal(rs[k], ps[k], err_msg=f"{seed} {k}")


def test_port_matches_reference_c2_sample(port, ref):
    b = W.c2_batch(duration_s=300.0, stride=41)
    cfg = lt.h100_like_config(1)
    r, _ = ref.simulate(b, cfg, sim_options(None, True))
    p, _ = port.simulate(b, cfg, sim_options(None, True))
    for f in r.dtype.names:
        if f not in SKIP:
            assert np.array_equal(r[f], p[f]), f


def test_port_matches_reference_errors(port, ref):
    cfg = lt.h100_like_config(8)
    cfg.load.cpu_load_seconds.pop(32)
    wls = [lt.WorkloadSpec([lt.AdapterSpec(1, 32, 0.5)], lt.LengthSpec.mean(100, 10, 50, 5), 60.0, 1),
           lt.WorkloadSpec([lt.AdapterSpec(1, 128, 0.5)], lt.LengthSpec.mean(100, 10, 50, 5), 60.0, 1),
           lt.WorkloadSpec([lt.AdapterSpec(1, 8, -1.0)], lt.LengthSpec.mean(100, 10, 50, 5), 60.0, 1),
           lt.WorkloadSpec([lt.AdapterSpec(1, 8, 1.0), lt.AdapterSpec(1, 8, 1.0)], lt.LengthSpec.mean(100, 10, 50, 5), 60.0, 1),
           lt.WorkloadSpec([lt.AdapterSpec(1, 8, 0.01)], lt.LengthSpec.mean(310000, 0, 20000, 0), 400.0, 3)]
    b = WorkloadBatch.from_workloads(wls, slots=[2, 64, 1, 1, 1])
    r, _ = ref.simulate(b, cfg, sim_options())
    p, _ = port.simulate(b, cfg, sim_options())
    np.testing.assert_array_equal(r["status"], p["status"])
    for i in range(len(wls)):
        assert ref.message(i) == port.message(i)


@pytest.mark.parametrize("profile", ["h100_like", "llama31_8b", "qwen25_7b"])
def test_profiles_parse_identically_in_the_reference(ref, profile):
    """The packaged server profiles (configs/*.json, the C5 workloads' llama31_8b
    and qwen25_7b) read by the reference's own server_config_from_json
    (json_io.cpp:188-235) equal what the ABI packs from them."""
    from paper_2508_08343_b200.batch import PackedConfig
    from paper_2508_08343_b200.types import profile_config
    path = os.path.join(os.path.dirname(lt.__file__), "configs", profile + ".json")
    for slots in (1, 32):
        rc, detail = ref.config_json_matches(open(path).read(), PackedConfig(profile_config(profile, slots)))
        assert rc == 1, detail
