"""bench.py's JSON-line contract on CPU: the reference arm (the reference's
own CPU path, oracle/_ref or the pinned port) on the small config prints one
parseable line with the keys the driver reads."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--config", "c1", "--steps", "3", "--warmup", "3"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "dtype", "config", "cpu_baseline", "e2e", "impl"):
        assert k in d, k
    assert d["impl"] == "reference" and d["steps"] == 3 and d["value"] > 0
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] == 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0


def test_both_arms_share_config_and_slice_bytes():
    """the reference arm and ours stream identical bytes and
    report the same `config` object; priming (graph-cache setup of our engine)
    is separate from the W warm-up updates and consumed by both arms."""
    import argparse
    import importlib.util
    import numpy as np
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    from paper_2308_16395_b200 import datagen as dg
    cfg = dg.CONFIGS["c2"]
    args = argparse.Namespace(config="c2")
    a = bench.base_config(args, cfg, "single")
    b = bench.base_config(args, cfg, "single")
    assert a == b and "numpy" in a["slice_source"] and a["n_slices"] == 100
    assert "slice_torch" in bench.slice_source(dg.CONFIGS["c4"])   # multi-GB slices: device synthesis
    small = dg.CONFIGS["c1"]
    gen = dg.make_stream(small)
    np.testing.assert_array_equal(bench.bench_slice_host(gen, small, 25), gen.slice_numpy(25))
