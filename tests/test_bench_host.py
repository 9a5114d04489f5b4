"""bench.py contract pieces that run without a GPU: the reference arm (CPU oracle) prints one JSON
line with the base keys and the same `config` object as our arm, and the roofline builder
returns the contract's fields."""
import json
import os
import subprocess
import sys

import bench
import synth_inputs as SI

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
             "scaling", "vs_baseline", "dtype", "data", "config"}


def test_reference_arm_json_line():
    import __graft_entry__
    __graft_entry__.build()   # a fresh checkout has no libsquares.so yet (the arm uses its keygen)
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "1"],
                       cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert BASE_KEYS <= set(d)
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["config"] == bench.config_for(SI.CONFIGS["c2"], 1, "weak")
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


def test_config_is_shared_and_scales():
    w = SI.CONFIGS["c2"]
    assert bench.config_for(w, 8, "weak")["samples_per_step"] == 8 * w.n
    assert bench.config_for(w, 8, "strong")["samples_per_step"] == w.n
    assert bench.config_for(SI.CONFIGS["c4"], 1, "weak")["samples_per_step"] == 4096 * (1 << 18)


def test_roofline_fields():
    peaks, src = bench.load_peaks()
    prof = bench.load_profile_summary()
    for name in ("c2", "c3", "c4", "c5"):
        w = SI.CONFIGS[name]
        rl = bench.roofline_for(w, {"ms_per_step": 1.0, "samples_rank": w.nkeys * w.n}, peaks, src, prof)
        assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= set(rl)
        assert abs(rl["frac"] - rl["achieved"] / rl["peak"]) < 1e-12
        if w.kind != "fused":
            assert rl["bound"] == "hbm" and rl["unit"] == "GB/s"
            assert rl["algorithmic_bytes_per_launch"] == w.nkeys * w.n * w.elem_bytes
        else:
            assert rl["bound"] == "alu" and rl["traffic"] is None
