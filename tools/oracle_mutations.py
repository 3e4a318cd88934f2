"""Mutation check of the oracle pins: apply each plausible
mistake to a scratch copy of oracle/ and require tests/test_oracle_pins.py to fail.

    python tools/oracle_mutations.py        # prints one line per mutation, exit 1 if one survives
    python tools/oracle_mutations.py --full # every mutation against the whole pin file (lists every catching pin)

By default each mutation is first run against the pin expected to catch it (HINTS) and
against the whole file only if that pin passes, so the check fits the CPU suite.
"""
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FULL = "--full" in sys.argv[1:]

MUTATIONS = {
    # Eq. 4 stabilisation term with the wrong sign (assembled matrix and row formula)
    "eq4_sign": [
        ("oracle/operator.py", 'return (-d2 * sp.identity(nA, format="csr") + (Dh + d2 * P) @ E).tocsr()',
         'return (d2 * sp.identity(nA, format="csr") + (Dh - d2 * P) @ E).tocsr()'),
        ("oracle/operator.py", "lap = -d2 * u_i + (nb - 6.0 * Eu_i) / h2 + d2 * Eu_i",
         "lap = d2 * u_i + (nb - 6.0 * Eu_i) / h2 - d2 * Eu_i"),
    ],
    "eq4_no_stabilisation": [
        ("oracle/operator.py", "lap = -d2 * u_i + (nb - 6.0 * Eu_i) / h2 + d2 * Eu_i",
         "lap = (nb - 6.0 * Eu_i) / h2"),
    ],
    # RAS: additive instead of restricted prolongation
    "ras_additive": [("oracle/ras.py", "z[d] = zj[self.keep[j]]", "z[o] += zj")],
    # overlap one layer short (reading R7)
    "overlap_layers_minus_1": [("oracle/ras.py", "for _ in range(layers):", "for _ in range(max(layers - 1, 0)):")],
    # FOM square solve instead of the GMRES least-squares problem (reading R6)
    "arnoldi_fom": [("oracle/krylov.py", "y, *_ = np.linalg.lstsq(H[: kk + 1, :kk], e1, rcond=None)",
                     "y = np.linalg.solve(H[:kk, :kk], e1[:kk])")],
    # transposed stencil offsets (x <-> z) in the extension
    "stencil_transposed": [("oracle/interp.py",
                            "vals = wx[:, OFFS[:, 0]] * wy[:, OFFS[:, 1]] * wz[:, OFFS[:, 2]]",
                            "vals = wx[:, OFFS[:, 2]] * wy[:, OFFS[:, 1]] * wz[:, OFFS[:, 0]]")],
    # Lagrange weight nodes shifted (stencil centred one cell off)
    "stencil_base_shift": [("oracle/interp.py", "base = fl.astype(np.int64) - 1", "base = fl.astype(np.int64)")],
    # GMRES: Givens rotation sign
    "givens_sign": [("oracle/krylov.py", "g[j + 1] = -sn[j] * g[j]", "g[j + 1] = sn[j] * g[j]")],
    # band radius sqrt(16) h instead of sqrt(17) h (reading R1)
    "band_radius": [("oracle/band.py", "return math.sqrt(17.0) * h", "return math.sqrt(16.0) * h")],
    # strict instead of closed tube |x - cp(x)| <= lambda
    "band_strict": [("oracle/band.py", "out.append(ijk[dist <= lam])", "out.append(ijk[dist < lam - 0.5 * h])")],
    # ghosts from 4 of the 6 neighbours only
    "ghost_neighbours": [("oracle/band.py", "cand = (active[:, None, :] + NEIGHBORS6[None, :, :]).reshape(-1, 3)",
                          "cand = (active[:, None, :] + NEIGHBORS6[None, :4, :]).reshape(-1, 3)")],
    # band order: y and z bits of the brick Morton key swapped (reading R8)
    "morton_axes": [("oracle/order.py",
                     "m = _interleave(bx + (1 << 16)) | (_interleave(by + (1 << 16)) << 1) | (_interleave(bz + (1 << 16)) << 2)",
                     "m = _interleave(bx + (1 << 16)) | (_interleave(bz + (1 << 16)) << 1) | (_interleave(by + (1 << 16)) << 2)")],
    # band order: x slowest instead of fastest inside a brick
    "brick_cell_order": [("oracle/order.py", "keys[n] = m * 512 + lz * 64 + ly * 8 + lx",
                          "keys[n] = m * 512 + lx * 64 + ly * 8 + lz")],
    # shifted operator without its c u term (Eq. 2)
    "shift_dropped": [("oracle/operator.py", "return c * u_i - lap", "return -lap"),
                      ("oracle/operator.py",
                       'return (c * sp.identity(band.nA, format="csr") - laplace_beltrami_matrix(band, E)).tocsr()',
                       'return (-laplace_beltrami_matrix(band, E)).tocsr()')],
    # Schnakenberg: v's reaction with the sign of u's cubic term (configs[4])
    "reaction_sign": [("oracle/reaction.py", "return p.gamma * (p.a - u + u2v), p.gamma * (p.b - u2v)",
                       "return p.gamma * (p.a - u + u2v), p.gamma * (p.b + u2v)")],
    # IMEX: the explicit term without its dt
    "imex_dt": [("oracle/reaction.py", "return c1 * (u + p.dt * ru), c2 * (v + p.dt * rv)",
                 "return c1 * (u + ru), c2 * (v + rv)")],
    # IMEX: the two diffusivities swapped
    "imex_mu_swapped": [("oracle/reaction.py", "A1 = (sp.diags(c1 * I) - L).tocsc()", "A1 = (sp.diags(c2 * I) - L).tocsc()")],
    # manufactured rhs with l^2 instead of l(l+1) (north_star)
    "rhs_eigenvalue": [("oracle/problems.py", "return (c + l * (l + 1)) * real_sph(l, m, cp_of(band, ijk))",
                        "return (c + l * l) * real_sph(l, m, cp_of(band, ijk))")],
    # restarted GMRES: the correction of a cycle added with the wrong sign
    "gmres_modified_gs": [("oracle/krylov.py", "w = w - H[i, j] * V[i]", "w = w + H[i, j] * V[i]")],
}


# the pin expected to catch each mutation: run first (-x); the whole file only if it passes
HINTS = {
    "eq4_sign": "offlattice_plane_golden_rows", "eq4_no_stabilisation": "offlattice_plane_golden_rows",
    "ras_additive": "ras_stationary_iteration", "overlap_layers_minus_1": "overlap_equals_graph_distance_ball",
    "arnoldi_fom": "arnoldi_fixed_minimises", "stencil_transposed": "reproduce_tricubics",
    "stencil_base_shift": "semidiscrete_2d_golden", "givens_sign": "gmres_dense_random_vs_lu",
    "band_radius": "band_matches_pure_python", "band_strict": "band_matches_pure_python",
    "ghost_neighbours": "band_matches_pure_python", "morton_axes": "order_key_hand_values",
    "brick_cell_order": "order_key_hand_values", "shift_dropped": "gmres_cpm_tiny_band",
    "reaction_sign": "schnakenberg_constant_state", "imex_dt": "schnakenberg_constant_state",
    "imex_mu_swapped": "schnakenberg_constant_state", "rhs_eigenvalue": "manufactured_solution_second_order",
    "gmres_modified_gs": "gmres_identity_one_iteration",
}


def _run_one(name, edits):
    with tempfile.TemporaryDirectory() as tmp:
        for d in ("tests", "seeded_inputs", "oracle"):
            shutil.copytree(os.path.join(ROOT, d), os.path.join(tmp, d), ignore=shutil.ignore_patterns("__pycache__"))
        shutil.copy(os.path.join(ROOT, "pytest.ini"), tmp)
        for f, a, b in edits:
            p = os.path.join(tmp, f)
            s = open(p).read()
            if a not in s:
                return name, None
            open(p, "w").write(s.replace(a, b))
        env = dict(os.environ, OMP_NUM_THREADS="1", OPENBLAS_NUM_THREADS="1", MKL_NUM_THREADS="1")
        cmd = [sys.executable, "-m", "pytest", "tests/test_oracle_pins.py", "-q", "-rf", "-p", "no:cacheprovider",
               "-m", "not gpu"]
        failed = []
        for extra in ((["-x", "-k", HINTS[name]],) if name in HINTS and not FULL else ()) + ([],):
            r = subprocess.run(cmd + extra, cwd=tmp, capture_output=True, text=True, env=env)
            failed = [ln.split("::")[1].split(" ")[0] for ln in r.stdout.splitlines() if ln.startswith("FAILED")]
            if failed:
                break
        return name, failed


def main() -> int:
    from concurrent.futures import ThreadPoolExecutor

    workers = max(1, min(len(MUTATIONS), (os.cpu_count() or 1) // (2 if FULL else 1)))
    with ThreadPoolExecutor(workers) as ex:
        results = list(ex.map(lambda kv: _run_one(*kv), MUTATIONS.items()))
    bad = 0
    for name, failed in results:
        if failed is None:
            print(f"{name}: anchor not found")
            bad = 1
        elif not failed:
            print(f"{name}: SURVIVED")
            bad = 1
        else:
            print(f"{name}: caught by {', '.join(failed)}")
    return bad


if __name__ == "__main__":
    sys.exit(main())
