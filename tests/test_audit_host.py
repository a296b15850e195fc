"""Host side of the audit / bench / CLI harness (paper_1502_05216_b200.audit,
cli, tables): the sample streams equal the reference's own (golden vectors made
by running pkg/src/twofold/audit.py:130-158, tests/golden/gen_audit_samples.py),
report types round-trip like the reference's, and the GPU entry points refuse
to run without a device (no CPU fallback)."""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

from paper_1502_05216_b200 import FUNCTION_NAMES, audit, cli, tables


@pytest.fixture(scope="module")
def streams():
    return dict(np.load(os.path.join(GOLDEN, "audit_samples.npz")))


@pytest.mark.parametrize("width", (64, 32))
@pytest.mark.parametrize("fn", FUNCTION_NAMES)
def test_sample_stream_matches_reference(fn, width, streams):
    u = np.uint64 if width == 64 else np.uint32
    for seed in (42, 0xB0B):
        x0, x1 = audit.gen_sample_arrays(audit.SampleSpec(fn, width, 256, seed))
        assert np.array_equal(x0.view(u), streams[f"{fn}_{width}_{seed}_x0"].view(u))
        assert np.array_equal(x1.view(u), streams[f"{fn}_{width}_{seed}_x1"].view(u))
    t = next(audit.gen_samples(audit.SampleSpec(fn, width, 1, 42)))
    assert t.value == float(streams[f"{fn}_{width}_42_x0"][0])


def test_thresholds_and_budget():
    assert audit.thresholds_for("texp", 64) == (2.0 ** -100, 2.0 ** -95)
    assert audit.thresholds_for("plog1p", 32) == (2.0 ** -42, 2.0 ** -36)
    assert audit.warn_budget_for(100_000) == 1
    assert audit.warn_budget_for(1_000_000) == 2
    assert audit.warn_budget_for(1_000_001) == 3
    assert "saturation" in audit.SampleSpec("texp", 64, 1, 1).domain


def test_report_json_roundtrip():
    r = audit.AccuracyReport(fn="tlog", width=64, backend="fma", etalon="oracle", samples=10,
                             seed=1, l1_rel=2.0 ** -105, l0_rel=2.0 ** -100, warnings=0,
                             thresholds={"l1": 2.0 ** -98, "l0": 2.0 ** -93, "warn_budget": 1},
                             subnormals_excluded=2)
    r.passed = audit.recompute_pass(r)
    assert r.passed
    d = json.loads(r.to_json())
    assert d["pass"] is True and "passed" not in d
    assert audit.AccuracyReport.from_json(r.to_json()) == r
    assert r.summary_line().endswith(": pass")
    b = audit.BenchReport(fn="texp", width=32, backend="fma", iterations=5, elapsed_seconds=1.0,
                          mops=2.0, baseline_mops=1.0, checksum="00ff", unreliable=False)
    assert audit.BenchReport.from_json(b.to_json()) == b
    assert "x2.00" in b.summary_line()


def test_run_accuracy_argument_errors():
    spec = audit.SampleSpec("texp", 64, 8, 1)
    with pytest.raises(ValueError):
        audit.run_accuracy(spec, etalon="mpfr")
    with pytest.raises(ValueError):
        audit.run_accuracy(spec, etalon="lib")
    with pytest.raises(ValueError):
        audit.run_accuracy(spec, oracle_precision=64)


def test_gpu_entry_points_fail_loudly_without_device():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError, match="no CUDA device"):
        audit.run_accuracy(audit.SampleSpec("texp", 64, 8, 1))
    with pytest.raises(RuntimeError, match="no CUDA device"):
        audit.run_bench("texp", 64, 100)


def test_cli_parser_and_tables(tmp_path):
    ap = cli.build_parser()
    a = ap.parse_args(["audit", "--fn", "all", "--width", "32", "--etalon", "lib"])
    assert a.samples == 100_000 and a.seed == 42 and a.etalon == "lib"
    b = ap.parse_args(["bench", "--fn", "texp"])
    assert b.iters == 200_000 and b.width == 64
    with pytest.raises(SystemExit):
        cli._fn_list("sin")
    assert len(cli._fn_list("all")) == 20
    assert cli.main(["tables", "--emit", str(tmp_path / "t{width}.txt"), "--width", "32"]) == 0
    text = (tmp_path / "t32.txt").read_text()
    assert text == tables.dump_tables(32)
    assert text.startswith("twofold-tables 1 width=32 L=1 K=5 N=6 Km1=7 Nm1=5 prec=192\n")


@pytest.mark.parametrize("width", (64, 32))
def test_table_dump_equals_reference_file(width):
    ref = f"/root/reference/pkg/src/twofold/data/tables_binary{width}.txt"
    if not os.path.exists(ref):
        pytest.skip("reference not mounted")
    assert tables.dump_tables(width) == open(ref).read()
    with pytest.raises(ValueError):
        tables.gen(width, 2 * (53 if width == 64 else 24) + 59)
