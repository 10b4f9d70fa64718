"""The HVP kernels and PCG run-time options against the oracle: MPL_HVP_KERNEL,
MPL_PCG_MAP, MPL_PDL and MPL_L2WIN are read once per process, so each case runs
tests/_hvp_variant_check.py in a subprocess.  Checks the HVP (and its elastic part), the Jacobi
diagonal and a replayed implicit step on a two-material scene with partially filled tiles, fp32 and
fp64, and the PSD-projected tangent."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CASES = [
    # (env, scene)
    ({"MPL_HVP_KERNEL": "wz"}, "mix_fp32"),
    ({"MPL_HVP_KERNEL": "wh"}, "mix_fp32"),
    ({"MPL_HVP_KERNEL": "wh"}, "psd_fp32"),
    ({"MPL_PCG_MAP": "group"}, "mix_fp32"),
    ({"MPL_PDL": "0", "MPL_L2WIN": "0"}, "mix_fp32"),
    ({"MPL_PCG_MAP": "warp"}, "mix_fp64"),
    # single-reduction PCG (the slab-rank default) on one GPU; classic is the one-GPU default
    ({"MPL_PCG": "cg1"}, "mix_fp32"),
    ({"MPL_PCG": "cg1", "MPL_CG1_E": "4"}, "mix_fp32"),
    ({"MPL_PCG": "cg1"}, "mix_fp64"),
    ({"MPL_PCG": "cg1"}, "psd_fp64"),
    # P2Q gather form (8 lanes per cell) vs the scatter default (tile-staged shared-memory accumulation)
    ({"MPL_P2Q": "gather"}, "mix_fp32"),
    ({"MPL_P2Q": "gather"}, "mix_fp64"),
    ({"MPL_P2Q": "gather"}, "watermix_fp64"),
    ({"MPL_P2Q": "gather"}, "vmmix_fp64"),
    ({"MPL_P2Q": "gather"}, "cfg1_fp32"),
    ({"MPL_P2Q": "gather"}, "cfg1b"),
    ({"MPL_SORT": "scatter"}, "mix_fp32"),   # the source-ordered sort (the gather form is default)
    ({"MPL_SORT": "scatter"}, "mix_fp64"),
    ({"MPL_KC": "0"}, "cfg1_fp32"),          # the 45-number tangent where the compressed one is the default
    ({"MPL_KC": "0"}, "cfg2s_fp32"),
    ({"MPL_KC_MINB": "4"}, "cfg2s_fp32"),   # 16 warps per SM (128 registers) instead of the default 12
    ({"MPL_KC_MINB": "3"}, "cfg2s_fp32"),   # ptxas capped at 148 registers (the default asks for 2 CTAs per SM: 168)
    ({"MPL_G2P": "particle"}, "mix_fp32"),   # one thread per particle with its own cell lookups (tile default)
    ({"MPL_G2P": "particle"}, "watermix_fp64"),
    ({"MPL_P2Q_HI": "1"}, "mix_fp32"),       # the dense-bucket P2Q kernel (default only at >= 40 particles per cell)
    ({"MPL_P2Q_HI": "1"}, "mix_fp64"),
    ({"MPL_P2Q_HI": "1"}, "cfg1_fp32"),
    # fp32 PCG vector kernels with the residual buffer holding r instead of the default z = D^-1 r
    ({"MPL_PCG_Z": "0"}, "mix_fp32"),
    ({"MPL_PCG_Z": "0"}, "psd_fp32"),
    ({"MPL_PCG_CPS": "8"}, "mix_fp32"),      # four waves of update CTAs instead of the one resident wave
    # two PCG iterations captured into a CUDA graph and replayed (device-side iteration index)
    ({"MPL_PCG_GRAPH": "1"}, "cfg1_fp32"),
    ({"MPL_PCG_GRAPH": "1"}, "cfg2s_fp32"),
    ({"MPL_PCG_GRAPH": "1"}, "psd_fp32"),
]


@pytest.mark.gpu
@pytest.mark.parametrize("env,scene", CASES, ids=[
    "-".join(f"{k[4:].lower()}={v}" for k, v in e.items()) + f"-{s}" for e, s in CASES])  # noqa: E501
def test_hvp_variant_parity(env, scene):
    e = dict(os.environ)
    for k in ("MPL_HVP_KERNEL", "MPL_PCG_MAP", "MPL_PDL", "MPL_L2WIN", "MPL_PCG", "MPL_CG1_E", "MPL_P2Q", "MPL_SORT",
              "MPL_KC", "MPL_KC_MINB", "MPL_G2P", "MPL_P2Q_HI", "MPL_PCG_Z", "MPL_PCG_CPS", "MPL_PCG_GRAPH"):
        e.pop(k, None)
    e.update(env)
    r = subprocess.run([sys.executable, "-m", "tests._hvp_variant_check", scene], cwd=ROOT, env=e,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert "OK" in r.stdout


@pytest.mark.gpu
def test_slab_ranks_with_classic_pcg():
    """The slab decomposition (loopback ranks) with the two-kernel PCG instead of the slab default
    (single-reduction): replayed step and multi-step migration parity (tests/test_gpu_slabs.py)."""
    e = dict(os.environ)
    e["MPL_PCG"] = "classic"
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "tests/test_gpu_slabs.py", "-k",
                        "replayed_step or migration_multistep_matches_one_rank"], cwd=ROOT, env=e,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


@pytest.mark.gpu
def test_slab_ranks_without_hvp_split():
    """Slab ranks with the HVP in one launch and the halo after it (MPL_OVERLAP=0) instead of the default
    split (interface tiles, halo, interior tiles): replayed step and multi-step migration parity."""
    e = dict(os.environ)
    e["MPL_OVERLAP"] = "0"
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "tests/test_gpu_slabs.py", "-k",
                        "replayed_step or migration_multistep_matches_one_rank"], cwd=ROOT, env=e,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
