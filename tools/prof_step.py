"""Small fixed workload for ncu: config-1 band, 3 applies, 60 GMRES(50) iterations."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2110_06322_b200 as cpm
import seeded_inputs

h = float(os.environ.get("CPM_H", 1.0 / 200))
band = cpm.cpm_build_band("sphere", h)
coords = cpm.cpm_band_active_coords(band).astype(np.int64)
u = torch.from_numpy(seeded_inputs.uniform_pm1(0, coords)).cuda()
y = torch.empty_like(u)
for _ in range(3):
    cpm.cpm_apply(band, 10.0, u, y)
f = torch.empty_like(u)
cpm.cpm_eval_sph(band, 6, 3, 52.0, f)
x = torch.zeros_like(u)
st = cpm.cpm_solve(band, 10.0, f, x, rtol=1e-10, restart=50, maxit=int(os.environ.get("CPM_MAXIT", 60)))
torch.cuda.synchronize()
print("nA", band.n, "its", st.iterations, "launches", cpm.cpm_kernel_launches())
