"""bench.py's CPU-side pieces: the reference arm (the oracle timed on host cores, the only place
bench.py may run oracle/) prints one JSON line with the contract's keys, and the kernel-name /
algorithmic-byte helpers match DESIGN §5."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "0"],
                       cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert "workload" in d["config"]


def test_hvp_helpers():
    import bench
    # 180 B of tangent per quadrature point + 28 B per active node (fp32), doubled in fp64
    assert bench.hvp_bytes(10, 20, 4) == 10 * 180 + 20 * 28
    assert bench.hvp_bytes(10, 20, 8) == 2 * (10 * 180 + 20 * 28)
    env = {k: os.environ.pop(k) for k in ("MPL_HVP_KERNEL",) if k in os.environ}
    try:
        assert bench.hvp_kernel_name(32) == "k_hvp_wz"
        assert bench.hvp_kernel_name(64) == "k_hvp_wh<double, 3>"
    finally:
        os.environ.update(env)
