"""The RAS set-up's layout switches (read once per process, so each variant runs in
a subprocess): segments padded to 32-element starts (CPM_RAS_ALIGN, the inner
reduction pass then runs the register-direct kernel) and the cells of Sigma_A
outside a subdomain filled from a zero buffer (CPM_RAS_ZRUNS) instead of cleared
boxes.  The zero-source fill stages the same boxes (bit-identical RAS apply); the
padding changes only the summation order of the inner dot products."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
import paper_2110_06322_b200 as cpm, seeded_inputs
band = cpm.cpm_build_band("torus", 0.05, R=1.0, r=0.4)
ga = cpm.cpm_band_active_coords(band).astype(np.int64)
r = torch.from_numpy(seeded_inputs.uniform_pm1(4, ga)).cuda()
ras = cpm.cpm_ras_setup(band, 8, 4, 12, 1.0)
z = torch.empty_like(r)
cpm.cpm_ras_apply(ras, r, z)
f = torch.empty_like(r)
cpm.cpm_eval_torus_rhs(band, seeded_inputs.smooth_modulation_coeffs(1), f)
x = torch.zeros_like(r)
st = cpm.cpm_solve(band, 1.0, f, x, rtol=1e-10, restart=30, ras=ras)
torch.cuda.synchronize()
np.save({out!r} + ".z.npy", z.cpu().numpy())
np.save({out!r} + ".x.npy", x.cpu().numpy())
print(st.iterations, int(st.converged))
"""


def _run(tmp_path, name, env):
    out = str(tmp_path / name)
    e = dict(os.environ)
    e.update(env)
    p = subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT, out=out)], env=e, capture_output=True,
                       text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    its, conv = map(int, p.stdout.split()[-2:])
    return np.load(out + ".z.npy"), np.load(out + ".x.npy"), its, conv


def test_ras_layout_variants(tmp_path):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    z11, x11, it11, c11 = _run(tmp_path, "a1z1", {"CPM_RAS_ALIGN": "1", "CPM_RAS_ZRUNS": "1"})
    z10, x10, it10, c10 = _run(tmp_path, "a1z0", {"CPM_RAS_ALIGN": "1", "CPM_RAS_ZRUNS": "0"})
    z01, x01, it01, c01 = _run(tmp_path, "a0z1", {"CPM_RAS_ALIGN": "0", "CPM_RAS_ZRUNS": "1"})
    assert c11 and c10 and c01
    # zero-source runs vs cleared boxes: the same boxes, the same arithmetic
    assert np.array_equal(z11, z10) and np.array_equal(x11, x10) and it11 == it10
    # padded vs unpadded segments: the inner dot products summed in another order
    assert np.abs(z11 - z01).max() <= 1e-10 * np.abs(z01).max()
    assert abs(it11 - it01) <= 1
    assert np.abs(x11 - x01).max() <= 1e-8 * np.abs(x01).max()
