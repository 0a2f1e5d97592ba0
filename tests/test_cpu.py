"""CPU-only checks (no GPU): the C-ABI library loads and exports every symbol
include/loratwin_gpu.h declares; the glibc libm ports and the MT19937-64 /
seed_seq restatement are bit-exact against the host's glibc / libstdc++; host
types follow the reference's semantics."""
import os
import re
import subprocess

import numpy as np
import pytest

import paper_2508_08343_b200 as lt
from paper_2508_08343_b200 import _abi as A
from paper_2508_08343_b200 import build as B
from tests.conftest import ROOT


def test_library_exports_every_declared_symbol():
    B.build_gpu()
    header = open(os.path.join(ROOT, "include", "loratwin_gpu.h")).read()
    declared = set(re.findall(r"^[A-Za-z_][\w \*]*?\b(lt_\w+)\(", header, re.M))
    assert len(declared) >= 15
    lib = lt.load_library()
    for name in declared:
        assert hasattr(lib.dll, name), name
    assert set("lt_" + k for k in A.SIGNATURES) == declared
    assert lib.abi_version() == A.ABI_VERSION


def test_device_group_argument_errors_without_a_gpu():
    import ctypes as C

    lib = lt.load_library()
    st = A.lt_status()
    assert not lib.create_devices(None, 0, C.byref(st))
    assert st.code == A.LT_ERR_VALIDATION and b"no devices" in st.message
    st = A.lt_status()
    assert not lib.create_mask(0, C.byref(st))
    assert st.code == A.LT_ERR_VALIDATION and b"empty device mask" in st.message
    assert lib.device_count(None) == 0 and lib.gather_transport(None) == A.GATHER_NONE


def test_reference_side_binding_builds_and_reports_no_device():
    """integration/gpu_backend.cpp (the shim INTEGRATION.md describes),
    compiled against the reference's own headers and linked with its TUs and
    libloratwin_gpu.so; without a GPU the library's LT_ERR_DEVICE status
    comes back as the reference's InternalError."""
    from oracle import pyoracle

    if not os.path.exists(pyoracle.SHIM_CHECK):
        if not os.path.isdir(pyoracle.REFERENCE_SRC):
            pytest.skip("built only where /root/reference exists")
        pyoracle.build("shim")
    p = subprocess.run([pyoracle.SHIM_CHECK], capture_output=True, text=True, timeout=120)
    if p.returncode == 0:
        pytest.skip("a GPU is visible: tests/test_gpu_report.py runs the full check")
    assert p.returncode == 3, p.stdout + p.stderr
    assert p.stdout.startswith("no-device: ")


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", B.LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_status_messages_match_reference_text():
    lib = lt.load_library()
    import ctypes as C
    buf = C.create_string_buffer(320)
    lib.format_status(2, 1, 128, 0, buf, 320)
    assert buf.value.decode() == "infeasible configuration: 128 slots consume the entire KV budget (mem_max = 0)"
    lib.format_status(3, 3, 42, 0, buf, 320)
    assert buf.value.decode() == "single request exceeds KV capacity: request 42"
    lib.format_status(2, 2, 64, 0, buf, 320)
    assert buf.value.decode() == "estimators.load.cpu_load_seconds: no entry for rank 64"


def test_libm_ports_bit_exact_vs_host_glibc():
    B.build_native()
    exe = os.path.join(B.NATIVE_BIN, "libm_check")
    res = subprocess.run([exe, "auto", "400000", "3"], capture_output=True, text=True)
    assert res.returncode == 0, res.stdout
    # and the other glibc build, forced through the tunable
    env = dict(os.environ, GLIBC_TUNABLES="glibc.cpu.hwcaps=-AVX2,-FMA,-FMA4,-AVX")
    res = subprocess.run([exe, "auto", "400000", "4"], capture_output=True, text=True, env=env)
    assert res.returncode == 0, res.stdout


def test_libm_boundary_regressions():
    """Inputs near the log1p branch point 0xbfd2bec4 (a strict '<' in the machine code)."""
    B.build_native()
    res = subprocess.run([os.path.join(B.NATIVE_BIN, "libm_check"), "auto", "50000", "13"],
                         capture_output=True, text=True)
    assert res.returncode == 0


def test_mt19937_64_seed_seq_pinned():
    B.build_native()
    res = subprocess.run([os.path.join(B.NATIVE_BIN, "rng_check")], capture_output=True, text=True)
    assert res.returncode == 0 and "OK" in res.stdout


def test_host_libm_variant_probe():
    v = lt.load_library().host_libm_variant()
    assert v in (0, 1)


def test_g_candidates_and_enumeration():
    # placement.cpp:159-167 / test_placement.cpp:147-158
    assert lt.SweepGrid(n_values=[8]).g_candidates(8) == [2, 4, 8]
    assert lt.SweepGrid(n_values=[1]).g_candidates(1) == [1]
    assert lt.SweepGrid(n_values=[64]).g_candidates(64) == [8, 16, 32, 64]
    g = lt.SweepGrid(n_values=[4], g_mode=lt.GMode.Explicit, g_values=[2, 4, 8, 16])
    assert g.g_candidates(4) == [2, 4]
    conds = lt.enumerate_conditions(list(range(10)), [8, 16, 32], lt.LengthSpec.mean(1, 0, 1, 0))
    assert len(conds) == 220 * 10
    assert [l.rate for l in conds[0].mix] == [0, 0, 0] and [l.rank for l in conds[1].mix] == [8, 8, 16]


def test_instantiate_condition_round_robin():
    c = lt.Condition(mix=[lt.AdapterTemplate(8, 0.1), lt.AdapterTemplate(32, 0.2)], lengths=lt.LengthSpec.mean(1, 0, 1, 0))
    w = lt.instantiate_condition(c, 5, 60.0, 3)
    assert [a.adapter_id for a in w.adapters] == [1, 2, 3, 4, 5]
    assert [a.rank for a in w.adapters] == [8, 32, 8, 32, 8]


def test_c2_vectorised_packing_matches_object_packing():
    from tests import workloads as W
    from paper_2508_08343_b200.batch import WorkloadBatch

    wls, slots = W.c2_workloads(duration_s=600.0, stride=5)
    a = WorkloadBatch.from_workloads(wls, slots=slots)
    b = W.c2_batch(duration_s=600.0, stride=5)
    for f in ("adapter_offset", "n_adapters", "duration_s", "seed", "slots", "n_requests"):
        np.testing.assert_array_equal(a.scenarios[f], b.scenarios[f])
    for f in ("adapter_id", "rank", "rate"):
        np.testing.assert_array_equal(a.adapters[f], b.adapters[f])
