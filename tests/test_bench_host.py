"""CPU checks of bench.py's host-side helpers (the GPU run itself is the
driver's): the live pipe fractions and the committed SASS / ncu summaries
they read."""
import importlib.util
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench():
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def test_pipe_fractions():
    b = _bench()
    p = b.pipe_fractions(1.0e11, 1965.0, "fp64", 148)
    sass = json.load(open(os.path.join(ROOT, "profiles", "sass_walk_step.json")))["fp64_ring"]
    assert abs(p["issue_frac"] - sass["instructions_per_step"] * 1e11 / (148 * 128 * 1965e6)) < 1e-12
    assert abs(p["fp64_pipe_frac"] - sass["fp64_per_step"] * 1e11 / (148 * 64 * 1965e6)) < 1e-12
    assert 0 < p["fp64_pipe_frac"] < p["issue_frac"] < 1
    assert b.pipe_fractions(1.0e11, None, "fp64", 148) is None  # no clock sample: no figure
    assert "fp64_pipe_frac" not in b.pipe_fractions(1.0e11, 1965.0, "fp32", 148)


def test_ncu_summary_fields():
    b = _bench()
    s = b.ncu_summary()
    assert s is not None
    assert 0 < s["issue_slots_busy_pct"] <= 100 and 0 < s["fp64_pipe_pct"] <= 100
    assert 100 < s["instructions_per_path_step"] < 400
    assert 15 < s["dram_bytes_per_walk"] < 40  # algorithmic 20 B per walk record
    assert 28 <= s["active_lanes_per_warp_instruction"] <= 32
