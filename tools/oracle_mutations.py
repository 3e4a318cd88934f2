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
    # torus closest point with the major radius in place of the minor one
    "torus_cp_radius": [("oracle/surfaces.py", "cp[:, 2] = (self.r * dz) / dn", "cp[:, 2] = (self.R * dz) / dn")],
    # torus distance to the core circle instead of the surface
    "torus_dist": [("oracle/surfaces.py", "dist = np.abs(dn - self.r)\n        bad = (rho == 0.0) | (dn == 0.0)",
                    "dist = np.abs(dn)\n        bad = (rho == 0.0) | (dn == 0.0)")],
    # interpolation nodes (-1, 0, 1, 2) shifted to (0, 1, 2, 3)
    "lagrange_nodes": [("oracle/interp.py", "TAU = np.array([-1.0, 0.0, 1.0, 2.0])", "TAU = np.array([0.0, 1.0, 2.0, 3.0])")],
    # 7-point Laplacian with a 5 on the diagonal
    "laplacian_diagonal": [("oracle/operator.py", "vals = [np.full(nA, -6.0 / h2)]", "vals = [np.full(nA, -5.0 / h2)]")],
    # real spherical harmonics without the sqrt(2) of m != 0
    "sph_normalisation": [("oracle/sph.py", "return math.sqrt(2.0) * K * P * np.cos(am * ph)", "return K * P * np.cos(am * ph)")],
    # cos and sin branches of +m / -m swapped
    "sph_branches": [("oracle/sph.py", "if m > 0:\n        return math.sqrt(2.0) * K * P * np.cos(am * ph)",
                      "if m < 0:\n        return math.sqrt(2.0) * K * P * np.cos(am * ph)")],
    # config-2 rhs with the poloidal and toroidal angles exchanged
    "torus_rhs_angles": [("oracle/problems.py", "return np.cos(3.0 * th) * np.sin(2.0 * ph) * mod",
                          "return np.cos(3.0 * ph) * np.sin(2.0 * th) * mod")],
    # poloidal angle about the z axis instead of the core circle
    "torus_theta": [("oracle/problems.py", "th = np.arctan2(cp[:, 2], rho - R)", "th = np.arctan2(cp[:, 2], rho)")],
    # config-3 rhs noise amplitude
    "noise_amplitude": [("oracle/problems.py", "+ 1e-3 * seeded_inputs.normal(seed, ijk)", "+ 1e-2 * seeded_inputs.normal(seed, ijk)")],
    # GMRES: tolerance relative to the initial residual of each cycle instead of ||b||
    "gmres_target": [("oracle/krylov.py", "        beta = float(np.linalg.norm(r))\n        if beta <= target:",
                      "        beta = float(np.linalg.norm(r))\n        target = rtol * beta\n        if beta <= target:")],
    # GMRES: restart from zero instead of the current iterate
    "gmres_restart_update": [("oracle/krylov.py", "        x = x + Z[:k].T @ y", "        x = Z[:k].T @ y")],
    # RAS: restriction of the residual to the disjoint part only (no overlap data)
    "ras_keep_shift": [("oracle/ras.py", "self.keep = [np.searchsorted(o, d) for o, d in zip(self.over, self.disjoint)]",
                        "self.keep = [np.minimum(np.searchsorted(o, d) + 1, len(o) - 1) for o, d in zip(self.over, self.disjoint)]")],
    # RAS subdomains as slabs of the lattice-key order instead of the band (Morton) order
    "ras_slab_order": [("oracle/ras.py", "perm = band_order(band.active)", "perm = np.arange(band.nA)")],
    # Schnakenberg initial state: v = b / (a + b) instead of b / (a + b)^2
    "initial_state_v": [("oracle/reaction.py", "vs = p.b / (p.a + p.b) ** 2", "vs = p.b / (p.a + p.b)")],
    # slab bounds rounded up
    "slab_bounds_ceil": [("oracle/order.py", "return [(s * n) // S for s in range(S + 1)]",
                          "return [-((-s * n) // S) for s in range(S + 1)]")],
    # sphere closest point without the radius
    "sphere_radius": [("oracle/surfaces.py", "cp = (self.R * x) / r[:, None]", "cp = x / r[:, None]")],
    # fractional offset measured from the wrong lattice node (t = ceil - s)
    "stencil_offset": [("oracle/interp.py", "t = s - fl", "t = 1.0 - (s - fl)")],
    # barycentric weights without their alternating sign
    "barycentric_sign": [("oracle/interp.py", "beta[j] = 1.0 / prod", "beta[j] = abs(1.0 / prod)")],
    # row formula: five of the six neighbours
    "apply_rows_neighbours": [("oracle/operator.py", "    for off in NEIGHBORS6:\n        nb = nb + Eu_at(rows_ijk + off[None, :])",
                               "    for off in NEIGHBORS6[:5]:\n        nb = nb + Eu_at(rows_ijk + off[None, :])")],
    # row formula: u instead of E u at the neighbours (no extension before the stencil)
    "apply_rows_no_extension": [("oracle/operator.py", "        nb = nb + Eu_at(rows_ijk + off[None, :])",
                                 "        nb = nb + u_of_ijk(rows_ijk + off[None, :])")],
    # assembled operator: Delta_h applied to u, not to E u
    "laplacian_without_E": [("oracle/operator.py",
                             'return (-d2 * sp.identity(nA, format="csr") + (Dh + d2 * P) @ E).tocsr()',
                             'return (-d2 * sp.identity(nA, format="csr") + (Dh[:, :nA] + d2 * P[:, :nA])).tocsr()')],
    # ghost columns indexed without the nA offset
    "ghost_index_offset": [("oracle/band.py", "return np.where(ia >= 0, ia, np.where(ig >= 0, ig + self.nA, -1))",
                            "return np.where(ia >= 0, ia, np.where(ig >= 0, ig, -1))")],
    # GMRES: an iteration counted per Gram-Schmidt column as well
    "gmres_its_count": [("oracle/krylov.py", "            w = A(Z[j])\n            its += 1", "            w = A(Z[j])\n            its += 2")],
    # GMRES: back substitution over the wrong triangle
    "gmres_back_substitution": [("oracle/krylov.py", "y[i] = (g[i] - np.dot(H[i, i + 1:k], y[i + 1:k])) / H[i, i]",
                                 "y[i] = (g[i] - np.dot(H[i + 1:k, i], y[i + 1:k])) / H[i, i]")],
    # FGMRES: update with the Krylov basis V instead of the preconditioned vectors Z
    "fgmres_update_basis": [("oracle/krylov.py", "        x = x + Z[:k].T @ y", "        x = x + V[:k].T @ y")],
    # overlap grown through all 26 neighbours (reading R7: 6-neighbour layers)
    "overlap_26": [("oracle/ras.py", "    for _ in range(layers):\n        grow = inside.copy()",
                    "    for _ in range(2 * layers):\n        grow = inside.copy()")],
    # IMEX: (c + Delta) instead of (c - Delta)
    "imex_operator_sign": [("oracle/reaction.py", "A2 = (sp.diags(c2 * I) - L).tocsc()", "A2 = (sp.diags(c2 * I) + L).tocsc()")],
    # IMEX: shift 1/dt instead of 1/(dt mu)
    "imex_shift": [("oracle/reaction.py", "    c1, c2 = 1.0 / (p.dt * p.mu1), 1.0 / (p.dt * p.mu2)\n    return c1 * (u + p.dt * ru)",
                    "    c1, c2 = 1.0 / p.dt, 1.0 / p.dt\n    return c1 * (u + p.dt * ru)")],
    # Schnakenberg noise amplitude
    "initial_noise": [("oracle/reaction.py", "return (us + 1e-2 * seeded_inputs.uniform_pm1(seed, ijk, stream=0),",
                       "return (us + 1e-1 * seeded_inputs.uniform_pm1(seed, ijk, stream=0),")],
    # interpolation weights where cp falls on a lattice node (t = 0): the unit vector is not substituted
    "interp_exact_node": [("oracle/interp.py", "    w[hit] = exact[hit].astype(np.float64)\n", "")],
    # fixed-step Arnoldi: happy breakdown one column short
    "arnoldi_breakdown_index": [("oracle/krylov.py", "            kk = j + 1\n            break", "            kk = j\n            break")],
    # Condon-Shortley phase left in (reading R9 removes it)
    "sph_condon_shortley": [("oracle/sph.py", "P = lpmv(am, l, ct) * (-1.0) ** am", "P = lpmv(am, l, ct)")],
    # Schnakenberg u-kinetics a + u - u^2 v
    "reaction_u_terms": [("oracle/reaction.py", "return p.gamma * (p.a - u + u2v), p.gamma * (p.b - u2v)",
                          "return p.gamma * (p.a + u - u2v), p.gamma * (p.b - u2v)")],
    # GMRES ignores the initial guess
    "gmres_x0_ignored": [("oracle/krylov.py", "x = np.zeros(n) if x0 is None else np.array(x0, dtype=np.float64)",
                          "x = np.zeros(n)")],
    # RAS: one more inner step than asked for
    "ras_kinner_plus_1": [("oracle/ras.py", "zj = arnoldi_fixed(lambda v, Aj=Aj: Aj @ v, rj, self.k)",
                           "zj = arnoldi_fixed(lambda v, Aj=Aj: Aj @ v, rj, self.k + 1)")],
    # RAS: local problems on the disjoint parts (block Jacobi) although the overlap is grown
    "ras_local_problem_disjoint": [("oracle/ras.py", "self.over = [grow_overlap(band, d, overlap) for d in self.disjoint]",
                                    "self.over = [d for d in self.disjoint]")],
    # stencil base by truncation instead of floor (wrong for negative coordinates)
    "stencil_trunc": [("oracle/interp.py", "fl = np.floor(s)", "fl = np.trunc(s)")],
    # grid box one node short (|i| <= M - 1)
    "grid_box_clip": [("oracle/band.py", "ihi = [min(M, int(math.ceil(hi[c] / h)) + 1) for c in range(3)]",
                       "ihi = [min(M - 1, int(math.ceil(hi[c] / h)) + 1) for c in range(3)]")],
    # the config-2 modulation subtracted instead of added (reading R10)
    "modulation_sign": [("oracle/problems.py", "mod = mod + a * np.sin(kx * cp[:, 0] + ky * cp[:, 1] + kz * cp[:, 2])",
                         "mod = mod - a * np.sin(kx * cp[:, 0] + ky * cp[:, 1] + kz * cp[:, 2])")],
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
    "torus_cp_radius": "torus_cp_matches_brute_force", "torus_dist": "band_matches_pure_python",
    "lagrange_nodes": "lagrange_weights_golden", "laplacian_diagonal": "delta_h_exact_on_quadratics",
    "sph_normalisation": "real_sph_orthonormal", "sph_branches": "real_sph_closed_forms",
    "torus_rhs_angles": "rhs_torus_symmetries", "torus_theta": "torus_angles_invert",
    "noise_amplitude": "rhs_noisy_sph_noise_level", "gmres_target": "gmres_dense_random_vs_lu",
    "gmres_restart_update": "gmres_dense_random_vs_lu", "ras_keep_shift": "ras_single_subdomain_exact",
    "ras_slab_order": "ras_subdomains_are_band_order_slabs", "initial_state_v": "initial_state_recipe",
    "slab_bounds_ceil": "partition_and_overlap_invariants",
    "sphere_radius": "sphere_cp_closed_form", "stencil_offset": "semidiscrete_2d_golden",
    "barycentric_sign": "lagrange_weights_golden", "apply_rows_neighbours": "semidiscrete_2d_golden",
    "apply_rows_no_extension": "semidiscrete_2d_golden", "laplacian_without_E": "constants_in_kernel",
    "ghost_index_offset": "delta_h_exact_on_quadratics", "gmres_its_count": "gmres_identity_one_iteration",
    "gmres_back_substitution": "gmres_dense_random_vs_lu", "fgmres_update_basis": "ras_fgmres_converges",
    "overlap_26": "overlap_equals_graph_distance_ball", "imex_operator_sign": "schnakenberg_pure_diffusion",
    "imex_shift": "schnakenberg_constant_state", "initial_noise": "initial_state_recipe",
    "interp_exact_node": "E_on_lattice_plane_is_selection", "sph_condon_shortley": "real_sph_closed_forms",
    "reaction_u_terms": "schnakenberg_steady_state", "arnoldi_breakdown_index": "arnoldi_fixed_happy_breakdown",
    "gmres_x0_ignored": "gmres_initial_guess", "modulation_sign": "rhs_torus_modulation",
    "ras_kinner_plus_1": "ras_inexact_local_solve_takes_k_steps", "grid_box_clip": "band_clipped_by_the_grid_box",
    "ras_local_problem_disjoint": "ras_stationary_iteration", "stencil_trunc": "reproduce_tricubics",
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
