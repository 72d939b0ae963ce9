"""bench.py's JSON line keeps the driver's contract (checked on the committed round-end line and
on bench.py's own argument parser; the line itself needs the B200)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _line():
    with open(os.path.join(ROOT, "profiles", "r01l_bench_default.json")) as fh:
        return json.loads(fh.read().splitlines()[0])


def test_bench_line_has_the_contract_keys():
    d = _line()
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e",
              "gpu_launches", "roofline", "cpu_baseline", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["warmup"] >= 3 and d["higher_is_better"] is True
    assert abs(d["value"] - 10_200_478 * d["steps"] / (d["ms_per_step"] * d["steps"] * 1e-3)) \
        <= 1e-6 * d["value"]
    assert d["config"]["workload"].startswith("c3") and "l2" in d["config"]
    r = d["roofline"]
    assert r["bound"] in ("hbm", "tensor", "fp32") and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    e = d["e2e"]
    assert e["unit"] == d["unit"] and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert 0 < e["value"] < d["value"]
    cb = d["cpu_baseline"]
    assert cb["kind"] in ("port", "reference") and cb["cores"] >= 1 and cb["value"] > 0
    assert d["clocks"]["sm_mhz"] and not (set(d["clocks"]["reasons"]) &
                                          {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"})
    assert d["gpu_launches"] > 0


def test_bench_cli_parses_the_driver_flags():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--help"],
                         capture_output=True, text=True, cwd=ROOT, timeout=120)
    assert out.returncode == 0
    for flag in ("--gpus", "--steps", "--warmup", "--impl", "--config", "--e2e-steps",
                 "--pi-block", "--graph"):
        assert flag in out.stdout, flag


def test_bench_py_compiles():
    """bench.py parses (the driver runs it as a script; --help above imports only argparse)."""
    import ast
    with open(os.path.join(ROOT, "bench.py")) as fh:
        ast.parse(fh.read())


@pytest.mark.gpu
def test_bench_default_legs_on_c1():
    """The whole default bench (tuning, timed steps, e2e, collapsed and FP64 legs, CPU baseline)
    end to end on the small C1 dam break, so a broken leg fails here, not at round end."""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", "c1",
                          "--steps", "5", "--warmup", "3", "--e2e-steps", "3",
                          "--collapsed-step", "50", "--fp64-steps", "2", "--cpu-budget-s", "2"],
                         capture_output=True, text=True, cwd=ROOT, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    d = json.loads(out.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "e2e", "roofline", "cpu_baseline", "collapsed", "fp64", "gpu_launches"):
        assert k in d, k
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["collapsed"]["value"] > 0
