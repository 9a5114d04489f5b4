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
    import oracle
    oracle.build()
    # the reference arm must never load the product library: run it with the library hidden
    env = dict(os.environ, SQ_LIB="/nonexistent/libsquares.so")
    prog = ("import sys, runpy; sys.argv = ['bench.py', '--impl', 'reference', '--steps', '1', '--warmup', '1'];"
            "runpy.run_path('bench.py', run_name='__main__');"
            "bad = [m for m in sys.modules if m.startswith('paper_2004_06278_b200')];"
            "maps = open('/proc/self/maps').read();"
            "assert not bad and 'libsquares' not in maps, ('reference arm loaded the product', bad)")
    r = subprocess.run([sys.executable, "-c", prog], cwd=ROOT, capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert BASE_KEYS <= set(d)
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["config"] == bench.config_for(SI.CONFIGS["c2"], 1, "strong")
    assert d["scaling"] == "strong"
    assert d["cpu_baseline"]["cpu_model"]
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


def test_config_is_shared_and_scales():
    """Strong scaling (the default) keeps BASELINE.json's fixed totals at every N; weak
    scaling is opt-in and multiplies them."""
    for name in ("c2", "c3", "c4", "c5"):
        w = SI.CONFIGS[name]
        for n in (1, 2, 4, 8):
            assert bench.config_for(w, n, "strong")["samples_per_step"] == w.nkeys * w.n
        assert bench.config_for(w, 8, "weak")["samples_per_step"] == 8 * w.nkeys * w.n
    import argparse
    ap_default = [a for a in open(os.path.join(ROOT, "bench.py")).read().split("\n") if '"--scaling"' in a]
    assert ap_default and 'default="strong"' in ap_default[0]


def test_cpu_baseline_one_core():
    """per-kind 1-core oracle rates with dead-code guards."""
    import oracle
    oracle.build()
    key = bench._oracle_keys(SI.CONFIGS["c2"], 1)[0]
    oc = bench.one_core_rates(key, window=1 << 14, reps=3)
    assert set(oc["rates"]) == {"u32", "u64", "f32", "fused", "u32_xorfold"}
    assert all(v["msamples_per_s"] > 0 for v in oc["rates"].values())
    assert bench.cpu_model()


def test_roofline_fields():
    peaks, src = bench.load_peaks()
    prof = bench.load_profile_summary()
    for name in ("c2", "c3", "c4", "c5"):
        w = SI.CONFIGS[name]
        rl = bench.roofline_for(w, {"ms_per_step": 1.0, "samples_rank": w.nkeys * w.n}, peaks, src, prof,
                                {name: {"instructions_per_sample": 1.0}})
        assert rl["sass"]["instructions_per_sample"] == 1.0
        assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= set(rl)
        assert abs(rl["frac"] - rl["achieved"] / rl["peak"]) < 1e-12
        if w.kind != "fused":
            assert rl["bound"] == "hbm" and rl["unit"] == "GB/s"
            assert rl["algorithmic_bytes_per_launch"] == w.nkeys * w.n * w.elem_bytes
        else:
            assert rl["bound"] == "alu" and rl["traffic"] is None


def test_sass_counts_cover_every_bench_line():
    """The SASS-per-sample counts bench.py embeds in each roofline (tools/sass_counts.py,
    cuobjdump, no GPU) find every hot loop of the built library, with plausible totals."""
    import shutil
    import pytest
    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump not available")
    import __graft_entry__
    __graft_entry__.build()
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import sass_counts
    d = sass_counts.per_workload()
    assert {"c2", "c2_devkeys", "c3", "c4", "c5"} <= set(d)
    for k, v in d.items():
        assert 8 <= v["instructions_per_sample"] <= 40, (k, v["instructions_per_sample"])
        assert v["mix_per_sample"].get("IMAD.WIDE.U32", 0) >= 1, k
    assert d["c5"]["mix_per_sample"].get("ATOMS.ADD") == 1.0
