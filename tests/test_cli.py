"""The sphbench-compatible CLI and benchmark harness (cli.py, harness.py).

Modelled on the reference's tests/test_cli.py: usage errors, config files and the exit-code
mapping run on the CPU (no device call is reached); ``run`` / ``bench`` end to end need the
B200 and are marked ``gpu``."""
import pytest

sph = pytest.importorskip("paper_1110_3711_b200")
from paper_1110_3711_b200 import cli, harness  # noqa: E402
from paper_1110_3711_b200.sim import DivergenceError  # noqa: E402
from paper_1110_3711_b200.snapshots import CompareReport, FieldDiff, read_snapshot, read_stats  # noqa: E402


def test_usage_error_exit_code(capsys):
    assert cli.main(["frobnicate"]) == cli.EXIT_USAGE
    assert cli.main(["run", "--engine", "warp"]) == cli.EXIT_USAGE
    assert cli.main(["run", "--dp", "0.03"]) == cli.EXIT_USAGE  # neither --steps nor --tend
    assert cli.main(["run", "--steps", "1", "--precision", "fp16"]) == cli.EXIT_USAGE
    assert cli.main(["run", "--steps", "1", "--pi-block", "64"]) == cli.EXIT_USAGE
    assert "error" in capsys.readouterr().err


def test_config_file_supplies_defaults(tmp_path):
    cfg = tmp_path / "bench.cfg"
    cfg.write_text("# comment\ndp = 0.03\nsteps = 2\nsymmetry = off\nverify = yes\n")
    args = cli.parse_args(["--config", str(cfg), "run"])
    assert args.dp == 0.03 and args.steps == 2 and args.symmetry == "off" and args.verify is True
    args = cli.parse_args(["--config", str(cfg), "run", "--dp", "0.05"])  # explicit flags win
    assert args.dp == 0.05
    bad = tmp_path / "bad.cfg"
    bad.write_text("dp 0.03\n")
    assert cli.main(["--config", str(bad), "run", "--steps", "1"]) == cli.EXIT_USAGE


def test_engine_config_from_flags():
    args = cli.parse_args(["run", "--steps", "1", "--engine", "gather", "--symmetry", "off",
                           "--gather-variant", "slowcellsh", "--precision", "fp64"])
    cfg = cli.engine_config_from(args)
    assert cfg.tag == "b200-gather-slowcellsh-fp64" and cfg.required_n_subdiv() == 1
    # the reference rejects symmetric gather (config.py validated()); so does the shim
    args = cli.parse_args(["run", "--steps", "1", "--engine", "gather"])
    assert cli.main(["run", "--steps", "1", "--engine", "gather"]) == cli.EXIT_USAGE
    with pytest.raises(ValueError):
        cli.engine_config_from(args)


def test_exit_code_mapping(monkeypatch):
    def boom_divergence(args):
        raise DivergenceError("gone", step=3, particle_id=7)

    monkeypatch.setattr(cli, "cmd_run", boom_divergence)
    assert cli.main(["run", "--steps", "1"]) == cli.EXIT_DIVERGENCE
    report = CompareReport(fields=[FieldDiff("vel", 1.0, 1.0, 3, False)], passed=False)

    def boom_equiv(args):
        raise harness.EquivalenceError("a", "b", report)

    monkeypatch.setattr(cli, "cmd_run", boom_equiv)
    assert cli.main(["run", "--steps", "1"]) == cli.EXIT_EQUIVALENCE


def test_equivalence_error_message_and_report_format(tmp_path):
    report = CompareReport(fields=[FieldDiff("pos", 0.0, 0.0, 1, True),
                                   FieldDiff("vel", 2.0, 0.5, 42, False)], passed=False)
    e = harness.EquivalenceError("base", "other", report)
    assert str(e) == "base vs other: field vel diverges by rel 5.000e-01 at particle id 42"
    assert e.report is report
    rows = [harness.BenchRow("a", 100, 4, 2.0, 2.0, 0.0, 10, 5, 10, 400),
            harness.BenchRow("b", 100, 4, 0.5, 8.0, 0.0, 10, 5, 10, 400)]
    harness.apply_speedups(rows, "a")
    assert [r.speedup for r in rows] == [1.0, 4.0]
    assert rows[1].particle_steps_per_second == 800.0
    rep = harness.BenchReport(rows=rows, baseline_tag="a")
    text = rep.format_table()
    assert "(* baseline: a)" in text and text.splitlines()[2].endswith(" *")
    rep.to_csv(tmp_path / "r.csv")
    lines = (tmp_path / "r.csv").read_text().splitlines()
    assert lines[0] == ",".join(harness.BenchRow.CSV_FIELDS) and len(lines) == 3
    assert rep.row("b").steps_per_second == 8.0
    with pytest.raises(KeyError):
        rep.row("c")


def test_run_benchmark_validates_matrix_before_running():
    sc = sph.Scenario(dp=0.03)
    prm = sph.make_params(sc)
    m = harness.device_matrix()
    assert len({c.tag for c in m}) == 6 and harness.DEFAULT_BASELINE in {c.tag for c in m}
    with pytest.raises(ValueError, match="duplicate"):
        harness.run_benchmark(m + m[:1], sc, prm, 2, 1, harness.DEFAULT_BASELINE)
    with pytest.raises(ValueError, match="not in the matrix"):
        harness.run_benchmark(m, sc, prm, 2, 1, "cellpairs-off-l1-single")
    with pytest.raises(ValueError, match="steps"):
        harness.run_benchmark(m, sc, prm, 0, 1, harness.DEFAULT_BASELINE)


# ------------------------------------------------------------------ on the B200
@pytest.mark.gpu
def test_run_command_writes_snapshots_and_stats(tmp_path, capsys):
    rc = cli.main(["run", "--dp", "0.03", "--steps", "4", "--snap-every", "2",
                   "--out", str(tmp_path / "out")])
    assert rc == 0
    out_dir = tmp_path / "out"
    assert read_snapshot(out_dir / "snapshot_final.csv").id.size > 0
    assert (out_dir / "snapshot_000002.csv").exists() and (out_dir / "snapshot_000004.csv").exists()
    stats = read_stats(out_dir / "stats.jsonl")
    assert [s["step"] for s in stats] == [0, 1, 2, 3]
    assert all(s["true_pairs"] > 0 for s in stats)
    assert "steps/s" in capsys.readouterr().out


@pytest.mark.gpu
def test_run_command_gather_cells_and_verify(capsys):
    assert cli.main(["run", "--dp", "0.03", "--steps", "2", "--cells", "h/2"]) == 0
    assert cli.main(["run", "--dp", "0.03", "--steps", "2", "--pi-block", "384"]) == 0
    assert cli.main(["run", "--dp", "0.03", "--steps", "2", "--engine", "gather", "--symmetry",
                     "off", "--gather-variant", "slowcellsh"]) == 0
    assert cli.main(["run", "--dp", "0.03", "--steps", "3", "--verify"]) == 0
    assert "verify: ok" in capsys.readouterr().out


@pytest.mark.gpu
def test_bench_command_end_to_end(tmp_path, capsys):
    rc = cli.main(["bench", "--dp", "0.03", "--steps", "2", "--warmup", "1", "--out",
                   str(tmp_path / "rep")])
    assert rc == 0
    out = capsys.readouterr().out
    assert "baseline" in out and "steps/s" in out
    lines = (tmp_path / "rep" / "report.csv").read_text().splitlines()
    assert lines[0].startswith("tag,") and len(lines) == 7  # header + 6 device configurations


@pytest.mark.gpu
def test_equivalence_gate_trips():
    sc = sph.Scenario(dp=0.03)
    prm = sph.make_params(sc)
    m = [c for c in harness.device_matrix() if c.gather_variant == "slowcellsh"]
    rep = harness.run_benchmark(m, sc, prm, steps=3, warmup=1, baseline_tag=harness.DEFAULT_BASELINE)
    assert rep.row(harness.DEFAULT_BASELINE).speedup == 1.0
    assert all(len(v) == 3 for v in rep.stats_by_tag.values())
    with pytest.raises(harness.EquivalenceError):  # FP32 vs FP64 states are not bit-equal
        harness.run_benchmark(m, sc, prm, steps=3, warmup=1, baseline_tag=harness.DEFAULT_BASELINE,
                              tolerances={"pos": 0.0, "vel": 0.0, "rho": 0.0, "press": 0.0})
