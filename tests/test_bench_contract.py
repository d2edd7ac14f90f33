"""bench.py's contract on the CPU: the reference arm's JSON line (the oracle timed on the host),
and the byte models the roofline fractions divide by, pinned to SURVEY.md §8(d)'s table."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from synth import get_config  # noqa: E402


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "1",
                          "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["metric"] == bench.METRIC
    assert d["unit"] == "variances/s" and d["higher_is_better"] is True and d["value"] > 0
    assert d["n_gpus"] == 1 and d["steps"] == 1 and d["warmup"] == 0 and d["vs_baseline"] is None
    assert d["config"]["workload"] == "cfg1_1d_fp64"
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    e = d["e2e"]
    assert e["value"] == d["value"] and e["unit"] == d["unit"]
    assert e["h2d_bytes_per_step"] == 0 and e["d2h_bytes_per_step"] == 0


@pytest.mark.parametrize("ci,gb", [(2, 44.2), (3, 23.0), (4, 95.0)])
def test_build_byte_model_matches_survey(ci, gb):
    """SURVEY.md §8(d) 'Targets' table: B_build (1 GPU) = 44.2 / 23.0 / 95.0 GB for cfg2-4."""
    p = get_config(ci)
    assert bench.build_bytes(p, p.n) / 1e9 == pytest.approx(gb, rel=0.01)


def test_cfg1_build_bytes_and_query_models():
    p = get_config(1)
    assert bench.build_bytes(p, p.n) / 1e6 == pytest.approx(24.0, rel=0.05)     # SURVEY: 24 MB
    # d = 3 gathered-row model: B_query = 4^d k s_R + 8d + s_out = 25,628 B (cfg4)
    p4 = get_config(4)
    qb, model = bench.query_bytes(p4, 100)
    assert qb == 25_628 and "gathered" in model
    # d <= 2 cell-block model: x* (8d), the packed fp64 block (10 / 136 values), the result
    p2, p3 = get_config(2), get_config(3)
    assert bench.query_bytes(p2, 100)[0] == 8 + 8 * 10 + 4
    assert bench.query_bytes(p3, 100)[0] == 16 + 8 * 136 + 4


def test_reorth_byte_model():
    """Dominant-kernel bytes: dots (j+1) n s_v + n s_v and update (j+1) n s_v + 2 n s_v per
    pass, summed over j = 0..k-1 (the last step has no update)."""
    n, k = 1_000_000, 100
    rb = bench.reorth_bytes(n, k, 4, 1)
    want = sum((j + 1) * n * 4 + n * 4 + (j + 1) * n * 4 + 2 * n * 4 for j in range(k - 1))
    assert sum(v for v in rb.values() if isinstance(v, int)) == want or rb.get("total") == want
