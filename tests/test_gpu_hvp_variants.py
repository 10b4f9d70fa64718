"""Every HVP kernel variant and layout option against the oracle: MPL_HVP_KERNEL,
MPL_KZ_PAD and MPL_PCG_MAP are read once per process, so each case runs tests/_hvp_variant_check.py in
a subprocess.  Checks the HVP (and its elastic part), the Jacobi diagonal and a replayed implicit step
on a two-material fp32 scene with partially filled tiles and an fp64 scene."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CASES = [
    # (env, scene)
    ({"MPL_HVP_KERNEL": "wz"}, "mix_fp32"),
    ({"MPL_HVP_KERNEL": "wz", "MPL_KZ_PAD": "1"}, "mix_fp32"),
    ({"MPL_HVP_KERNEL": "wz2"}, "mix_fp32"),
    ({"MPL_HVP_KERNEL": "wzp"}, "mix_fp32"),
    ({"MPL_HVP_KERNEL": "wzs"}, "mix_fp32"),
    ({"MPL_HVP_KERNEL": "wzs2"}, "mix_fp32"),
    ({"MPL_HVP_KERNEL": "wz3"}, "mix_fp32"),
    ({"MPL_HVP_KERNEL": "wh"}, "mix_fp32"),
    ({"MPL_HVP_KERNEL": "wh4"}, "mix_fp32"),
    ({"MPL_HVP_KERNEL": "rp10"}, "mix_fp32"),
    ({"MPL_HVP_KERNEL": "rq"}, "mix_fp32"),
    ({"MPL_HVP_KERNEL": "pipe2"}, "mix_fp32"),
    ({"MPL_HVP_KERNEL": "pipe3"}, "mix_fp32"),
    ({"MPL_HVP_KERNEL": "reg"}, "mix_fp32"),
    ({"MPL_PCG_MAP": "group"}, "mix_fp32"),
    ({"MPL_PDL": "0", "MPL_L2WIN": "0"}, "mix_fp32"),
    ({"MPL_HVP_KERNEL64": "sel", "MPL_HVP_KERNEL": "rp10"}, "mix_fp64"),
    ({"MPL_HVP_KERNEL64": "sel", "MPL_HVP_KERNEL": "pipe3"}, "mix_fp64"),
    ({"MPL_HVP_KERNEL64": "sel", "MPL_HVP_KERNEL": "rq"}, "mix_fp64"),
    ({"MPL_PCG_MAP": "warp"}, "mix_fp64"),
]


@pytest.mark.gpu
@pytest.mark.parametrize("env,scene", CASES, ids=[
    "-".join(f"{k[4:].lower()}={v}" for k, v in e.items()) + f"-{s}" for e, s in CASES])  # noqa: E501
def test_hvp_variant_parity(env, scene):
    e = dict(os.environ)
    for k in ("MPL_HVP_KERNEL", "MPL_HVP_KERNEL64", "MPL_KZ_PAD", "MPL_PCG_MAP", "MPL_PDL", "MPL_L2WIN"):
        e.pop(k, None)
    e.update(env)
    r = subprocess.run([sys.executable, "-m", "tests._hvp_variant_check", scene], cwd=ROOT, env=e,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert "OK" in r.stdout
