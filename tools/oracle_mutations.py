"""Mutation check of the oracle pins: apply each plausible
mistake to a scratch copy of oracle/ and require tests/test_oracle_pins.py to fail.

    python tools/oracle_mutations.py        # prints one line per mutation, exit 1 if one survives
"""
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

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
        r = subprocess.run([sys.executable, "-m", "pytest", "tests/test_oracle_pins.py", "-q", "-rf",
                            "-p", "no:cacheprovider", "-m", "not gpu"],
                           cwd=tmp, capture_output=True, text=True, env=env)
        return name, [ln.split("::")[1].split(" ")[0] for ln in r.stdout.splitlines() if ln.startswith("FAILED")]


def main() -> int:
    from concurrent.futures import ThreadPoolExecutor

    workers = max(1, min(len(MUTATIONS), (os.cpu_count() or 1) // 2))
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
