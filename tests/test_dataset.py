"""Batched generate_dataset (SURVEY 8f row 1; placement.cpp:100-137, :266-527).

CPU: the host pieces (condition_hash, encode_workload) against the compiled
reference. GPU: the dataset CSV written through lt_generate_dataset must be
byte-identical to the reference's generate_dataset on the same spec, including
resume after a torn tail and per-condition failure messages.
"""
import os

import pytest

import paper_2508_08343_b200 as lt
from paper_2508_08343_b200 import api


def small_spec(**kw):
    spec = lt.DatasetSpec(rates=[3.2, 0.4, 0.05], ranks=[8, 32], triple_size=2, condition_stride=1,
                          lengths=lt.LengthSpec.mean(250, 50, 231, 50), duration_s=90.0, seed=11,
                          grid=lt.SweepGrid(n_values=[1, 2, 4, 8, 16]),
                          sweep=lt.SweepOptions(early_exit=True, early_exit_k=2))
    for k, v in kw.items():
        setattr(spec, k, v)
    return spec


def hash_cases():
    conds = lt.enumerate_conditions([3.2, 0.4, 0.05, 0.003125], [8, 16, 32], lt.LengthSpec.mean(250, 50, 231, 50),
                                    triple_size=3, condition_stride=7)
    conds.append(lt.Condition(mix=conds[1].mix, lengths=lt.LengthSpec.full([(10, 20), (30, 40), (55, 7)])))
    conds.append(lt.Condition(mix=[lt.AdapterTemplate(0, 1e-9)], lengths=lt.LengthSpec.mean(23, 5, 27, 5)))
    grids = [lt.SweepGrid(n_values=[1, 2, 4, 8]), lt.SweepGrid(n_values=[3, 6, 96], g_mode=lt.GMode.Explicit,
                                                                  g_values=[2, 64, 4])]
    return conds, grids


def test_condition_hash_and_features_match_reference(ref):
    lib = lt.load_library()
    conds, grids = hash_cases()
    for c in conds:
        assert api.encode_workload(c, lib=lib) == api.encode_workload(c, lib=ref.lib)
        for g in grids:
            for dur, seed in ((600.0, 5), (123.456, 2 ** 63 + 7)):
                assert api.condition_hash(c, dur, seed, g, lib=lib) == api.condition_hash(c, dur, seed, g, lib=ref.lib)


def test_encode_workload_empty_mix_error(ref):
    with pytest.raises(lt.ValidationError, match="condition.mix: must be non-empty"):
        api.encode_workload(lt.Condition(mix=[], lengths=lt.LengthSpec.mean(1, 0, 1, 0)))


def _both(dev, ref, spec, cfg, tmp_path, name, prepare=None):
    paths = [os.path.join(tmp_path, f"{name}_gpu.csv"), os.path.join(tmp_path, f"{name}_ref.csv")]
    errs = [[], []]
    progs = []
    for k, (lib, ctx) in enumerate(((dev.lib, dev.ctx), (ref.lib, None))):
        if prepare:
            prepare(paths[k])
        progs.append(api.run_generate_dataset(lib, ctx, spec, cfg, paths[k], errs[k].append))
    data = [open(p, "rb").read() for p in paths]
    return data, errs, progs


@pytest.mark.gpu
def test_dataset_csv_matches_reference(dev, ref, tmp_path):
    data, errs, progs = _both(dev, ref, small_spec(), lt.h100_like_config(1), str(tmp_path), "plain")
    assert data[0] == data[1]
    assert errs[0] == errs[1]
    assert (progs[0].total_conditions, progs[0].completed, progs[0].failed) == \
           (progs[1].total_conditions, progs[1].completed, progs[1].failed)
    assert data[0].count(b"\n") == 1 + progs[0].completed


@pytest.mark.gpu
def test_dataset_resume_torn_tail_and_failures(dev, ref, tmp_path):
    """Resume from a file holding the first rows plus a torn line; without a
    rank-32 load latency, conditions with a rank-32 leg fail at their first
    load (estimators.cpp:79-81) and are reported in canonical order."""
    spec = small_spec(grid=lt.SweepGrid(n_values=[1, 4, 8], g_mode=lt.GMode.Explicit, g_values=[2, 4]))
    cfg = lt.h100_like_config(1)
    cfg.load.cpu_load_seconds.pop(32)
    full, _, _ = _both(dev, ref, spec, cfg, str(tmp_path), "full")
    assert full[0] == full[1]
    lines = full[1].split(b"\n")
    head = b"\n".join(lines[:3]) + b"\n" + lines[3][: len(lines[3]) // 2]

    def torn(p):
        with open(p, "wb") as f:
            f.write(head)

    data, errs, progs = _both(dev, ref, spec, cfg, str(tmp_path), "resume", torn)
    assert data[0] == data[1]
    assert errs[0] == errs[1] and len(errs[0]) == progs[0].failed > 0
    assert progs[0].completed == progs[1].completed


@pytest.mark.gpu
def test_dataset_full_mode_and_stride(dev, ref, tmp_path):
    spec = small_spec(lengths=lt.LengthSpec.full([(120, 40), (300, 90), (64, 200), (20, 10)]),
                      sweep=lt.SweepOptions(early_exit=False, mode=lt.LengthMode.Full), condition_stride=2,
                      rates=[1.6, 0.1, 0.0125])
    data, errs, _ = _both(dev, ref, spec, lt.h100_like_config(1), str(tmp_path), "fullmode")
    assert data[0] == data[1]
    assert errs[0] == errs[1]


@pytest.mark.gpu
def test_dataset_spec_errors_match_reference(dev, ref, tmp_path):
    cfg = lt.h100_like_config(1)
    for bad in (small_spec(triple_size=0), small_spec(rates=[]), small_spec(grid=lt.SweepGrid(n_values=[4, 2]))):
        msgs = []
        for lib, ctx in ((dev.lib, dev.ctx), (ref.lib, None)):
            with pytest.raises(lt.ValidationError) as e:
                api.run_generate_dataset(lib, ctx, bad, cfg, os.path.join(str(tmp_path), "x.csv"))
            msgs.append(str(e.value))
        assert msgs[0] == msgs[1]
