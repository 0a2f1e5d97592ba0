"""Robustness of the device path at its own limits:

  * the glibc libm ports as the device runs them (nvcc, sm_100a,
    --fmad=false) against the host glibc over 10^9 inputs per function
    (tests/native/libm_device.cu), in the reference's RNG domains (~12 s;
    10^10 per function is recorded in profiles/r2_sanitizer.txt);
  * the adapter-count limit of the engine's 1,024-bit lane masks
    (kMaxAdapters): 1,024 adapters run and match the reference, 1,025 are
    refused per scenario (LT_ERR_UNSUPPORTED) without failing the batch;
  * many-adapter batches on the 12-warp occupancy variant, whose per-warp
    shared memory must still fit the block (warps per block are dropped).
"""
import os
import subprocess

import numpy as np
import pytest

import paper_2508_08343_b200 as lt
from paper_2508_08343_b200 import _abi as A
from paper_2508_08343_b200.batch import WorkloadBatch, sim_options
from tests import workloads as W
from tests.conftest import ROOT

pytestmark = pytest.mark.gpu

LIBM_DEVICE = os.path.join(ROOT, "tests", "native", "bin", "libm_device")


def test_libm_ports_on_device_bit_exact_1e9_per_function():
    if not os.path.exists(LIBM_DEVICE):
        pytest.skip("tests/native/bin/libm_device not built")
    p = subprocess.run([LIBM_DEVICE, "auto", "1000000000", "7"], capture_output=True, text=True, timeout=900)
    lines = dict(l.split(None, 1) for l in p.stdout.strip().splitlines() if not l.startswith(" "))
    assert p.returncode == 0, p.stdout + p.stderr
    for fn in ("log1p", "log", "sin", "cos"):
        n, bad = map(int, lines[fn].split())
        assert n == 1_000_000_000 and bad == 0, (fn, n, bad)


def many_adapter_batch(ns, rate_total=2.0, duration=30.0):
    wls = []
    for i, n in enumerate(ns):
        ads = [lt.AdapterSpec(k + 1, (8, 16, 32)[k % 3], rate_total / n) for k in range(n)]
        wls.append(lt.WorkloadSpec(adapters=ads, lengths=lt.LengthSpec.mean(250, 50, 231, 50), duration_s=duration,
                                   seed=900 + i))
    return WorkloadBatch.from_workloads(wls, slots=[min(n, 64) for n in ns])


FIELDS = ("status", "iterations", "finished_count", "rejected_count", "preemptions", "load_events",
          "tokens_in_window", "starved", "digest", "final_clock_s", "throughput_tok_s")


@pytest.mark.parametrize("variant", ["1", "3"])
def test_adapter_limit_1024_and_1025(dev, ref, monkeypatch, variant):
    monkeypatch.setenv("LT_ENGINE_VARIANT", variant)
    batch = many_adapter_batch([1024, 1025, 640, 8])
    cfg = lt.h100_like_config(64)
    g, _ = dev.simulate_batch(batch, cfg, want_digest=True)
    r, _ = ref.simulate(batch, cfg, sim_options(None, True))
    assert int(g["status"][1]) == A.LT_ERR_UNSUPPORTED
    assert "at most 1024 adapters" in dev.message(1)
    for i in (0, 2, 3):
        for f in FIELDS:
            assert g[f][i] == r[f][i], (variant, i, f, g[f][i], r[f][i])
    assert int(g["iterations"][0]) > 0


def test_many_adapter_batch_on_occupancy_variant(dev, ref, monkeypatch):
    """Twelve 640-adapter engines with the 12-warp variant forced: 12 x
    (24 B x 640 + tables) exceeds the opt-in block budget, so the plan must
    fall back to fewer warps per block instead of failing the launch."""
    monkeypatch.setenv("LT_ENGINE_VARIANT", "3")
    batch = many_adapter_batch([640] * 12, rate_total=1.0, duration=20.0)
    cfg = lt.h100_like_config(64)
    g, _ = dev.simulate_batch(batch, cfg, want_digest=True)
    r, _ = ref.simulate(batch, cfg, sim_options(None, True))
    for f in FIELDS:
        np.testing.assert_array_equal(g[f], r[f], err_msg=f)


def test_check_invariants_passes_and_changes_nothing(dev, ref):
    """SimOptions.check_invariants runs the checked engine build (the
    reference's check_scheduler_invariants before every emit): clean runs
    give the unchecked results, fuzz engines with preemption included."""
    batch, cfg = W.summary_cases()
    a, sa = dev.simulate_batch(batch, cfg, want_states=True, want_digest=True)
    b, sb = dev.simulate_batch(batch, cfg, lt.SimOptions(check_invariants=True), want_states=True, want_digest=True)
    for f in FIELDS + ("status", "rejected_count"):
        np.testing.assert_array_equal(a[f], b[f], err_msg=f)
    for k in sa:
        np.testing.assert_array_equal(sa[k], sb[k], err_msg=k)
    for seed in range(12):
        ads, reqs, fcfg = W.scripted_fuzz(seed, n_requests=40 + seed % 50, n_adapters=1 + seed % 6)
        fb = WorkloadBatch.from_workloads([W.scripted_workload(ads, 6.0)], scripted=[reqs])
        g, _ = dev.simulate_batch(fb, fcfg, lt.SimOptions(check_invariants=True), want_digest=True)
        r, _ = ref.simulate(fb, fcfg, sim_options(lt.SimOptions(check_invariants=True), True))
        for f in ("status", "iterations", "digest", "preemptions"):
            assert g[f][0] == r[f][0], (seed, f)


def test_check_invariants_reports_a_ledger_fault(dev, monkeypatch):
    """A ledger fault injected on the device (test hook) is caught by the
    checked build and reported with the reference's InternalError text."""
    batch, cfg = W.summary_cases()
    monkeypatch.setenv("LT_INVARIANT_INJECT", "3")
    out, _ = dev.simulate_batch(batch, cfg, lt.SimOptions(check_invariants=True))
    hit = [i for i in range(len(out)) if int(out["status"][i]) == A.LT_ERR_INTERNAL]
    assert hit, "no engine reported the injected fault"
    msg = dev.message(hit[0])
    assert msg.startswith("KV ledger out of balance: holds sum to "), msg
    held, ledger = [int(t.strip(",")) for t in msg.split() if t.strip(",").isdigit()]
    assert ledger == held + 1
    monkeypatch.delenv("LT_INVARIANT_INJECT")
    clean, _ = dev.simulate_batch(batch, cfg, lt.SimOptions(check_invariants=True))
    assert (clean["status"] == A.LT_OK).sum() >= (out["status"] == A.LT_OK).sum()
