"""Golden fixtures for the field-of-values diagnostics (tests/golden/fov.npz),
made by running the REFERENCE (markovmg/fov.py, read-only at
/root/reference/pkg/src) in the build container.  The committed npz is what
tests/test_gpu_fov.py reads on any machine.

Usage:  OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden_fov.py

Per case: the input matrix, and the reference's fov_boundary (hull, sorted
eigenvalues, nu, contains_origin), eigenvalue_dots, project_range and
projected_preconditioned outputs.  Matrices: the reference's own test inputs
(tests/test_fov.py) plus chain matrices up to the dense cap's size class.
"""

from __future__ import annotations

import sys
import time
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
OUT = Path(__file__).resolve().parent / "fov.npz"
sys.path.insert(0, REF)
from markovmg import chains, fov, presets, solver  # noqa: E402
from markovmg.bootstrap import run_setup  # noqa: E402


def circulant_walk(n):
    A = np.zeros((n, n))
    for j in range(n):
        A[(j + 1) % n, j] = 0.5
        A[(j - 1) % n, j] = 0.5
    return np.eye(n) - A


def cases():
    rng = np.random.default_rng(0)
    S = rng.standard_normal((20, 20))
    yield "sym20", 0.5 * (S + S.T), 64
    yield "eye6", np.eye(6), 32
    yield "uniform8", chains.uniform_2d(8).B.toarray(), 64
    yield "tandem7", chains.tandem_queue(7).B.toarray(), 128
    yield "tandem6", chains.tandem_queue(6).B.toarray(), 64
    yield "circ12", circulant_walk(12), 64
    rng = np.random.default_rng(2)
    A = rng.standard_normal((30, 30)) * 0.1 + np.diag(2.0 + rng.random(30))
    yield "diag30", A, 64
    yield "diag30inv", np.linalg.inv(A), 64
    yield "bd40", chains.birth_death(40, 0.9).B.toarray(), 32
    rng = np.random.default_rng(5)
    yield "rand50", rng.standard_normal((50, 50)), 64
    yield "uniform16", chains.uniform_2d(16).B.toarray(), 64
    yield "tandem20", chains.tandem_queue(20).B.toarray(), 64
    yield "tandem34", chains.tandem_queue(34).B.toarray(), 32


def main():
    store = {}
    names = []
    for name, A, angles in cases():
        t = time.time()
        f = fov.fov_boundary(A, n_angles=angles)
        store[f"{name}_A"] = np.asarray(A, dtype=np.float64)
        store[f"{name}_angles"] = np.int64(angles)
        store[f"{name}_boundary"] = f.boundary
        store[f"{name}_eigenvalues"] = f.eigenvalues
        store[f"{name}_nu"] = np.float64(f.nu)
        store[f"{name}_inside"] = np.bool_(f.contains_origin)
        store[f"{name}_seconds"] = np.float64(time.time() - t)
        names.append(name)
        print(f"{name}: n={A.shape[0]} hull={f.boundary.size} nu={f.nu:.3e} inside={f.contains_origin} "
              f"{time.time() - t:.2f}s", flush=True)
    store["names"] = np.array(names)
    # project_range (fov.py:194-207)
    for name, p in (("bd30", chains.birth_death(30, 0.9)), ("uniform6", chains.uniform_2d(6))):
        t = time.time()
        pr = fov.project_range(p.B)
        store[f"pr_{name}_A"] = p.B.toarray()
        store[f"pr_{name}_basis"] = pr.basis
        store[f"pr_{name}_projected"] = pr.projected
        f = fov.fov_boundary(pr.projected, n_angles=64)
        store[f"pr_{name}_boundary"] = f.boundary
        store[f"pr_{name}_nu"] = np.float64(f.nu)
        store[f"pr_{name}_seconds"] = np.float64(time.time() - t)
        print(f"project_range {name}: rank {pr.basis.shape[1]} {time.time() - t:.2f}s", flush=True)
    # projected_preconditioned with the reference's own V-cycle (test_fov.py:108-116;
    # n = 289 is a single-level hierarchy, n = 1089 a three-level one)
    for n in (289, 1089):
        p = presets.build_problem("uniform2d", n=n)
        cfg = presets.default_setup_config("uniform2d", cycles=1, seed=1)
        res = run_setup(p, cfg)
        op = solver.VCycleOperator(res.hierarchy, cfg.smoother)
        t = time.time()
        pp = fov.projected_preconditioned(p.B, op)
        f = fov.fov_boundary(pp.projected, n_angles=64)
        key = f"pp_uniform{n}"
        store[f"{key}_levels"] = np.array([lev.n for lev in res.hierarchy.levels])
        if n <= 300:  # larger projections are pinned through their spectrum and FOV only
            store[f"{key}_projected"] = pp.projected
            store[f"{key}_basis"] = pp.basis
        store[f"{key}_rank"] = np.int64(pp.basis.shape[1])
        store[f"{key}_boundary"] = f.boundary
        store[f"{key}_eigenvalues"] = f.eigenvalues
        store[f"{key}_nu"] = np.float64(f.nu)
        store[f"{key}_inside"] = np.bool_(f.contains_origin)
        store[f"{key}_seconds"] = np.float64(time.time() - t)
        print(f"projected_preconditioned uniform{n}: levels {[lev.n for lev in res.hierarchy.levels]} "
              f"nu={f.nu:.4e} {time.time() - t:.2f}s", flush=True)
    np.savez_compressed(OUT, **store)
    print("wrote", OUT, OUT.stat().st_size, "bytes")


if __name__ == "__main__":
    main()
