"""The single-kernel (fused) apply experiment (apply.cu k_apply_fused, build.cu
build_fused): a band built with CPM_FUSED=1 evaluates E u for
its own eval nodes and its halo nodes in one kernel, with no E u round trip through
HBM.  Every node's contraction and the 7-point sum keep the split kernels' order,
so the result must equal the split apply bit for bit, and the oracle to 1e-12."""
import os

import numpy as np
import pytest

import seeded_inputs

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle.band import Band as OBand  # noqa: E402
from oracle.operator import shifted_operator  # noqa: E402
from oracle.surfaces import Sphere, Torus  # noqa: E402


@pytest.fixture(scope="module")
def cpm():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2110_06322_b200._build import build

    build()
    import paper_2110_06322_b200 as p

    return p


def _fused_band(cpm, kind, h, **kw):
    os.environ["CPM_FUSED"] = "1"
    try:
        return cpm.cpm_build_band(kind, h, **kw)
    finally:
        del os.environ["CPM_FUSED"]


@pytest.mark.parametrize("kind,h,kw", [("sphere", 0.1, {}), ("torus", 0.05, {"R": 1.0, "r": 0.4}),
                                       ("sphere", 0.06, {"R": 0.7})])
def test_fused_apply_equals_split_and_oracle(cpm, kind, h, kw):
    gs = cpm.cpm_build_band(kind, h, **kw)
    gf = _fused_band(cpm, kind, h, **kw)
    ga = cpm.cpm_band_active_coords(gs).astype(np.int64)
    assert np.array_equal(ga, cpm.cpm_band_active_coords(gf))
    u = torch.from_numpy(seeded_inputs.uniform_pm1(0, ga)).cuda()
    ys, yf = torch.empty_like(u), torch.empty_like(u)
    cpm.cpm_apply(gs, 3.0, u, ys)
    cpm.cpm_apply(gf, 3.0, u, yf)
    torch.cuda.synchronize()
    assert torch.equal(ys, yf)
    ob = OBand(Sphere(kw.get("R", 1.0)) if kind == "sphere" else Torus(kw["R"], kw["r"]), h)
    perm = ob.index_active(ga)
    uo = np.empty(ob.nA)
    uo[perm] = u.cpu().numpy()
    yo = (shifted_operator(ob, 3.0) @ uo)[perm]
    assert np.abs(yf.cpu().numpy() - yo).max() <= 1e-12 * np.abs(yo).max()
