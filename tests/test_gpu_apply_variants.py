"""The apply's A/B switches (read once per process, so each variant runs in a
subprocess) compute the same numbers: the fill with 8 or 4 lanes per run
(CPM_FILL), the extend's register / occupancy configurations (CPM_NT_CFG), the
pair dealing and stride choice (CPM_DEAL), the fill-run order (CPM_RUNSORT), the
per-element or TMA-fed laplace (CPM_LAP_TMA), PDL on or off (CPM_PDL): every node's
arithmetic is the same, so the applies are bit-identical."""
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
out = []
for kind, h, kw in [("sphere", 0.05, {{}}), ("torus", 0.04, {{"R": 1.0, "r": 0.4}})]:
    band = cpm.cpm_build_band(kind, h, **kw)
    ga = cpm.cpm_band_active_coords(band).astype(np.int64)
    u = torch.from_numpy(seeded_inputs.uniform_pm1(0, ga)).cuda()
    y = torch.empty_like(u)
    cpm.cpm_apply(band, 3.0, u, y)
    torch.cuda.synchronize()
    out.append(y.cpu().numpy())
np.save({out!r}, np.concatenate(out))
"""

VARIANTS = {
    "default": {},
    "fill8": {"CPM_FILL": "0"},
    "cfg8x3": {"CPM_NT_CFG": "0"},
    "cfg9x3": {"CPM_NT_CFG": "2"},
    "deal0": {"CPM_DEAL": "0"},
    "deal1": {"CPM_DEAL": "1"},
    "runsort0": {"CPM_RUNSORT": "0"},
    "laplace_elem": {"CPM_LAP_TMA": "0"},
    "nopdl": {"CPM_PDL": "0"},
}


def test_apply_variants_bit_identical(tmp_path):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    res = {}
    for name, env in VARIANTS.items():
        out = str(tmp_path / f"{name}.npy")
        e = dict(os.environ)
        e.update(env)
        p = subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT, out=out)], env=e,
                           capture_output=True, text=True, timeout=600)
        assert p.returncode == 0, (name, p.stderr[-2000:])
        res[name] = np.load(out)
    for name, y in res.items():
        assert np.array_equal(y, res["default"]), name
