"""bench.py's output contract: one JSON line carrying the driver's keys plus `roofline`,
`cpu_baseline` and `e2e`.  The committed round lines are checked here; on a GPU the smallest
BASELINE config is benchmarked live in a subprocess (stages 1-2 + evaluation, a few ms)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE = ["metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
        "scaling", "vs_baseline", "dtype", "data", "config", "e2e"]


def _check_line(d, reference=False):
    for k in BASE:
        assert k in d, k
    # BASELINE.json's metric is a triple ("lattice-sum+RHOSVD wall ms; grid-eval Gpts/s; % of
    # ... roofline"): `metric` is its first member, `grid_eval` and `roofline` carry the others
    assert json.load(open(os.path.join(ROOT, "BASELINE.json")))["metric"].startswith(d["metric"] + ";")
    assert d["unit"] == "ms" and d["higher_is_better"] is False and d["dtype"] == "f64"
    assert isinstance(d["config"], dict) and "workload" in d["config"] and "model" not in d["config"]
    assert d["vs_baseline"] is None  # BASELINE.md holds no published number for this metric
    e = d["e2e"]
    for k in ("value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"):
        assert k in e, k
    c = d["cpu_baseline"]
    if reference:
        assert d["impl"] == "reference" and e["h2d_bytes_per_step"] == 0 and e["d2h_bytes_per_step"] == 0
        assert c is not None and c["value"] == d["value"] == e["value"]
    if c is not None:
        for k in ("value", "unit", "cores", "kind", "sample"):
            assert k in c, k
        assert c["kind"] in ("port", "reference") and c["cores"] >= 1
    if not reference:
        r = d["roofline"]
        for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
            assert k in r, k
        assert r["bound"] in ("hbm", "tensor") and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-12
        assert d["gpu_launches"] > 0
        assert e["d2h_bytes_per_step"] > 0 and e["value"] >= d["value"]
        for k in ("sm_mhz", "sm_max_mhz", "reasons"):
            assert k in d["clocks"], k


def _last_json(path):
    return json.loads([ln for ln in open(path) if ln.startswith("{")][-1])


def test_committed_round_lines_follow_the_contract():
    d = _last_json(os.path.join(ROOT, "profiles", "bench_default_r02_final.json"))
    _check_line(d)
    assert d["config"]["workload"] == "cfg4" and d["n_gpus"] == 1
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["value"] > 1000 * d["value"] / 100
    r = _last_json(os.path.join(ROOT, "profiles", "bench_reference_r02_final.json"))
    _check_line(r, reference=True)
    assert r["config"] == d["config"]  # both arms describe one workload


@pytest.mark.gpu
def test_live_bench_line_on_the_smallest_config():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", "1", "--steps", "3",
                          "--warmup", "3", "--no-cpu"], capture_output=True, text=True, timeout=600,
                         env={**os.environ, "BENCH_NO_CLOCKS": ""})
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    _check_line(d)
    assert d["config"]["workload"] == "cfg1" and d["steps"] == 3 and d["warmup"] == 3
