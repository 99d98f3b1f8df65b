"""bench.py's reference arm (this tier's reference is the oracle) on the CPU:
one JSON line with the contract's keys, impl = "reference", a cpu_baseline
describing the run and an e2e with zero transfer bytes.  A bounded sample
(2 z-planes of config 4, init + 1 IRLS step)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "1", "--ref-planes", "2", "--ref-T", "1"],
                         check=True, capture_output=True, text=True, cwd=ROOT, timeout=900).stdout
    lines = [l for l in out.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["e2e"]["value"] == d["value"] and "workload" in d["config"]


@__import__("pytest").mark.gpu
def test_native_arm_json_line():
    """The GPU arm on config 2 (short run): every key of the contract, a
    roofline of the dominant kernel, e2e with its transfer bytes, clocks and
    the launch count."""
    import pytest
    try:
        import torch
        if not torch.cuda.is_available():
            pytest.skip("no CUDA device")
    except ImportError:
        pytest.skip("no torch")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", "config2", "--steps", "1",
                          "--warmup", "3", "--no-two-level", "--no-cpu-baseline", "--no-fixed-point-exit",
                          "--e2e-steps", "1"], check=True, capture_output=True, text=True, cwd=ROOT,
                         timeout=900).stdout
    lines = [l for l in out.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] < 2 and r["achieved"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0 and d["e2e"]["value"] > 0
    assert d["gpu_launches"] > 0 and d["value"] > 0 and d["config"]["cg_iters_per_step"] > 0
