"""Full-size (BASELINE.json configs 1-4) parity fixtures, made by running the REFERENCE.

Like make_golden.py this imports the upstream reference (`markovmg`, read-only
at /root/reference/pkg/src) and runs ONLY its own functions; it is the
generator of committed fixtures, never imported by tests or the product.

    python tests/golden/make_golden_big.py cfg1 cfg2 cfg4 cfg3 [--workers 6]

What runs, per config (BASELINE.json:configs[1..4]):
  * the chain: the reference's own generators `uniform_2d` / `tandem_queue`
    (chains.py:95-179); cfg3's Delaunay edge set comes from scipy's Qhull
    (the reference's Bowyer-Watson, chains.py:186-268, is O(n^2): weeks at
    2^21) and A is assembled from it exactly as chains.py:291-302 and
    validated by the reference's `_finish` (chains.py:39-61);
  * test vectors: BASELINE's uniform(0,1) seed-0 draws injected through the
    same `UniformShim` as make_golden.py (bootstrap.py:187-188);
  * `run_setup` (bootstrap.py:395-429) unmodified, except that the per-fine-
    point loop of `_build_rows` (interp.py:252-289) is spread over forked
    worker processes: every worker calls the reference's own `_build_rows`
    on the full level with the fine set restricted to its chunk, and the
    fitted rows are merged through the reference's `csr_from_coo`.  Fits
    are independent per point, so the merged operator is the serial one.
    Workers run single-threaded OpenBLAS (same LAPACK path as a serial run);
  * then `VCycleOperator` + `gmres` (solver.py:79-226) with rtol 1e-8 (cfg4:
    max_iters 120 -- the reference preallocates max_iters + 1 basis vectors).

Limits of this container (62 GB RAM, no GPU), recorded in each fixture:
  * cfg4's coarsest level has n_L = 16,384 after the reference's own
    `_operator_degenerate` truncation; `coarsest_triplets` builds the
    doubled 32,768^2 generalized eigenproblem (bootstrap.py:205-281,
    dense.py:74-92), whose numpy eigh peaks near 69 GB.  The coarsest
    TRIPLETS are therefore replaced by the incoming (smoothed, restricted)
    test vectors -- every splitting and every P / Q / B_l / M_l / N_l is
    built on the downward pass BEFORE that call and is the reference's
    own.  x0 is then not the reference's, so the solve is pinned from the
    uniform start x = 1/n on both sides (`gmres_start = "uniform"`): the
    reference's own V-cycle (with its SVD PinvOperator of B_L) and GMRES.
  * cfg3's coarsest (n_L = 47,824 expected) needs a 95,648^2 eigenproblem
    and a 47,824^2 SVD: the run stops at the coarsest call, so cfg3 pins
    every splitting and operator pattern of the downward pass only.

What is stored (compact; full x only for cfg1/cfg2):
  per operator: shape, nnz, sha256 of indptr and of indices (int64 bytes),
  value checksums (sum, sum|v|, projection on default_rng(12345) normals);
  per split: n, n_coarse, sha256 of the coarse index list;
  weights and sigmas (k doubles each); x: full (cfg1/cfg2) or every 64th
  entry plus 4096 block sums (cfg4); iterations, residual history, times.
"""

from __future__ import annotations

import argparse
import hashlib
import multiprocessing as mp
import sys
import time
import types
from pathlib import Path

import numpy as np
from scipy import sparse as sp
from threadpoolctl import threadpool_limits

REF = "/root/reference/pkg/src"
OUT = Path(__file__).resolve().parent

sys.path.insert(0, REF)
sys.path.insert(0, str(OUT))
from markovmg import bootstrap, chains, interp, presets, solver  # noqa: E402
from markovmg import sparse as msparse  # noqa: E402

from make_golden import UniformShim  # noqa: E402

CONFIGS = {
    # name: (family, side / n, k, gmres restart, what is pinned)
    "cfg1": ("uniform2d", 1023, 8, None, "full"),
    "cfg2": ("tandem", 1024, 16, 30, "full"),
    "cfg3": ("planar", 2 ** 21, 12, None, "downward"),
    "cfg4": ("tandem", 4095, 16, None, "uniform_start"),
}

_JOB = None
FIT_CPU = [0.0]
FIT_WALL = [0.0]


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(np.asarray(a, dtype=np.int64)).tobytes()).hexdigest()


def csr_sig(prefix, M, store):
    M = sp.csr_array(M)
    store[prefix + "_shape"] = np.asarray(M.shape, dtype=np.int64)
    store[prefix + "_nnz"] = np.int64(M.nnz)
    store[prefix + "_sha_indptr"] = np.asarray(sha(M.indptr))
    store[prefix + "_sha_indices"] = np.asarray(sha(M.indices))
    proj = np.random.default_rng(12345).standard_normal(M.nnz)
    store[prefix + "_vsum"] = np.asarray([M.data.sum(), np.abs(M.data).sum(), proj @ M.data])


def vec_sig(prefix, x, store, full=False):
    x = np.asarray(x, dtype=np.float64)
    store[prefix + "_blocks"] = np.add.reduceat(x, np.linspace(0, x.size, 4097).astype(np.int64)[:-1])
    store[prefix + "_every64"] = x[::64].copy()
    store[prefix + "_l1"] = np.float64(np.abs(x).sum())
    if full:
        store[prefix] = x


def _fit_chunk(chunk):
    B, split, tests, cfg, constrain = _JOB
    part = types.SimpleNamespace(coarse=split.coarse, fine=chunk, n=split.n,
                                 coarse_rank=split.coarse_rank, n_coarse=split.n_coarse)
    t0 = time.process_time()
    M = interp._build_rows(B, part, tests, cfg, constrain)
    M = sp.csr_array(M)
    keep = np.zeros(M.shape[0], dtype=bool)
    keep[chunk] = True
    rows = np.repeat(np.arange(M.shape[0]), np.diff(M.indptr))
    sel = keep[rows]
    return rows[sel], M.indices[sel], M.data[sel], time.process_time() - t0


def parallel_rows(B, split, tests, cfg, constrain, workers):
    """interp._build_rows with its fine-point loop spread over forked workers."""
    global _JOB
    _JOB = (B, split, tests, cfg, constrain)
    chunks = [c for c in np.array_split(np.asarray(split.fine), workers * 4) if c.size]
    t0 = time.perf_counter()
    with mp.get_context("fork").Pool(workers) as pool:
        parts = pool.map(_fit_chunk, chunks, chunksize=1)
    FIT_WALL[0] += time.perf_counter() - t0
    FIT_CPU[0] += sum(p[3] for p in parts)
    _JOB = None
    rows = np.concatenate([np.asarray(split.coarse)] + [p[0] for p in parts])
    cols = np.concatenate([np.arange(split.n_coarse)] + [p[1] for p in parts])
    vals = np.concatenate([np.ones(split.n_coarse)] + [p[2] for p in parts])
    return msparse.csr_from_coo(rows, cols, vals, (B.shape[0], split.n_coarse))


class CoarsestReached(Exception):
    pass


def build_chain(fam, size):
    if fam == "uniform2d":
        return chains.uniform_2d(size)
    if fam == "tandem":
        return chains.tandem_queue(size)
    from scipy.spatial import Delaunay
    n = size
    rng = np.random.default_rng(np.random.SeedSequence(1))  # chains.py:279-280
    pts = rng.random((n, 2))
    s = Delaunay(pts).simplices
    e = np.unique(np.sort(np.concatenate([s[:, [0, 1]], s[:, [1, 2]], s[:, [0, 2]]]), axis=1), axis=0)
    a, b = e[:, 0], e[:, 1]
    deg = np.bincount(a, minlength=n) + np.bincount(b, minlength=n)
    rows = np.concatenate([b, a])
    cols = np.concatenate([a, b])
    vals = np.concatenate([1.0 / deg[a], 1.0 / deg[b]])
    A = msparse.csr_from_coo(rows, cols, vals, (n, n))
    return chains._finish(A, "planar", {"n": n}, geometry=pts, seed=1)


def run(name, workers):
    fam, size, k, restart, mode = CONFIGS[name]
    store = {}
    t_gen = time.perf_counter()
    prob = build_chain(fam, size)
    t_gen = time.perf_counter() - t_gen
    n = prob.n
    csr_sig("B", prob.B, store)
    cfg = presets.default_setup_config(fam, cycles=1, seed=0, n_tests=k)
    # unrestarted GMRES preallocates max_iters + 1 basis vectors (solver.py:175):
    # the default 1000 is 125 GiB at cfg4; the solve converges in < 100
    # iterations, so a cap of 120 gives the identical iteration sequence
    gcfg = solver.GmresConfig(restart=restart, rtol=1e-8,
                              max_iters=120 if name == "cfg4" else solver.GmresConfig().max_iters)
    print(f"{name}: n={n} nnz={prob.B.nnz} built in {t_gen:.1f}s", flush=True)

    rec = {"entry": [], "split": [], "P": [], "Q": [], "Bc": [], "vw": [], "uw": [], "sigmas": []}
    orig = {k_: getattr(bootstrap, k_) for k_ in
            ("make_splitting", "singular_test_weights", "build_interpolation", "build_restriction",
             "triple_product", "bootstrap_cycle", "coarsest_triplets", "init_test_vectors",
             "_smooth_block")}

    def rec_cycle(B, M, N, trips, cfg_, geometry=None, depth=0, first_cycle=True, seed_stream=None):
        rec["entry"].append((B, M, N))
        print(f"  level {depth}: n={B.shape[0]} nnz={B.nnz} t={time.perf_counter() - T0:.0f}s", flush=True)
        return orig["bootstrap_cycle"](B, M, N, trips, cfg_, geometry, depth, first_cycle, seed_stream)

    def rec_split(B, geometry, ccfg, seed=None):
        s = orig["make_splitting"](B, geometry, ccfg, seed)
        rec["split"].append(s)
        return s

    def rec_stw(B, vectors, transpose_side=False, infinite_slot=None):
        t = orig["singular_test_weights"](B, vectors, transpose_side, infinite_slot)
        rec["uw" if transpose_side else "vw"].append(t.weights.copy())
        return t

    def par_interp(B, split, tests, icfg):
        P = parallel_rows(B, split, tests, icfg, False, workers)
        rec["P"].append(P)
        return P

    def par_restrict(B, split, tests, icfg):
        W = parallel_rows(msparse.transpose(B), split, tests, icfg,
                          icfg.constrain_constant_in_q, workers)
        Q = msparse.make_csr(msparse.transpose(W))
        rec["Q"].append(Q)
        return Q

    def rec_tp(Q, B, P, drop_tol=0.0):
        C = orig["triple_product"](Q, B, P, drop_tol)
        rec["Bc"].append(C)
        return C

    def rec_sb(B, diag, M, N, trips, cfg_, inhomogeneous):
        orig["_smooth_block"](B, diag, M, N, trips, cfg_, inhomogeneous)
        rec["sigmas"].append((B.shape[0], bool(inhomogeneous), trips.sigmas.copy()))

    def init(B, cfg_, rng=None):
        return orig["init_test_vectors"](B, cfg_, UniformShim(0, cfg_.n_tests, B.shape[0]))

    coarsest_info = {}

    def coarsest(B, M, N, r):
        coarsest_info["n"] = B.shape[0]
        if mode == "full":
            return orig["coarsest_triplets"](B, M, N, r)
        if mode == "downward":
            raise CoarsestReached()
        # uniform_start: the incoming triplets of this level (see module doc)
        trips = rec_cycle_trips[-1]
        return bootstrap.TripletSet(trips.sigmas.copy(), trips.left.copy(), trips.right.copy())

    rec_cycle_trips = []

    def rec_cycle2(B, M, N, trips, cfg_, geometry=None, depth=0, first_cycle=True, seed_stream=None):
        rec_cycle_trips.append(trips)
        return rec_cycle(B, M, N, trips, cfg_, geometry, depth, first_cycle, seed_stream)

    bootstrap.make_splitting = rec_split
    bootstrap.singular_test_weights = rec_stw
    bootstrap.build_interpolation = par_interp
    bootstrap.build_restriction = par_restrict
    bootstrap.triple_product = rec_tp
    bootstrap.bootstrap_cycle = rec_cycle2
    bootstrap.coarsest_triplets = coarsest
    bootstrap.init_test_vectors = init
    bootstrap._smooth_block = rec_sb
    FIT_CPU[0] = FIT_WALL[0] = 0.0
    T0 = time.perf_counter()
    setup = None
    try:
        with threadpool_limits(1):
            try:
                setup = bootstrap.run_setup(prob, cfg)
            except CoarsestReached:
                pass
    finally:
        for k_, f in orig.items():
            setattr(bootstrap, k_, f)
    t_setup = time.perf_counter() - T0
    print(f"{name}: setup {t_setup:.0f}s (fits: wall {FIT_WALL[0]:.0f}s, cpu {FIT_CPU[0]:.0f}s)", flush=True)

    for i, (B, M, N) in enumerate(rec["entry"]):
        csr_sig(f"E{i}_B", B, store)
        csr_sig(f"E{i}_M", M, store)
        csr_sig(f"E{i}_N", N, store)
    store["n_entries"] = np.int64(len(rec["entry"]))
    for i, s in enumerate(rec["split"]):
        store[f"S{i}_meta"] = np.asarray([s.n, s.n_coarse], dtype=np.int64)
        store[f"S{i}_sha"] = np.asarray(sha(s.coarse))
    store["n_splits"] = np.int64(len(rec["split"]))
    for key in ("P", "Q", "Bc"):
        for i, M in enumerate(rec[key]):
            csr_sig(f"{key}{i}", M, store)
        store[f"n_{key}"] = np.int64(len(rec[key]))
    for key in ("vw", "uw"):
        for i, w in enumerate(rec[key]):
            store[f"{key}{i}"] = w
    for i, (nl, inh, s) in enumerate(rec["sigmas"]):
        store[f"sm{i}_meta"] = np.asarray([nl, int(inh)], dtype=np.int64)
        store[f"sm{i}_sigmas"] = s
    store["n_smooth"] = np.int64(len(rec["sigmas"]))
    store["coarsest_n"] = np.int64(coarsest_info.get("n", -1))
    store["mode"] = np.asarray(mode)
    times = {"gen_s": t_gen, "setup_s": t_setup, "fit_wall_s": FIT_WALL[0], "fit_cpu_s": FIT_CPU[0],
             "workers": workers}

    if setup is not None:
        store["n_levels"] = np.int64(setup.hierarchy.depth)
        o_g, o_c, depth = bootstrap.complexities(setup.hierarchy)
        store["complexities"] = np.asarray([o_g, o_c, depth])
        vec_sig("x0", setup.x0, store)
        t1 = time.perf_counter()
        with threadpool_limits(8):
            vop = solver.VCycleOperator(setup.hierarchy, cfg.smoother)
        t_pinv = time.perf_counter() - t1
        x_init = setup.x0 if mode == "full" else np.full(n, 1.0 / n)
        store["gmres_start"] = np.asarray("x0" if mode == "full" else "uniform")
        t2 = time.perf_counter()
        with threadpool_limits(1):
            rep = solver.gmres(prob.B, np.zeros(n), x_init, gcfg, precond=vop)
        t_solve = time.perf_counter() - t2
        x = solver._sign_fix_l1(rep.x)
        vec_sig("x", x, store, full=(mode == "full"))
        store["iterations"] = np.int64(rep.iterations)
        store["history"] = np.asarray(rep.residual_history)
        store["converged"] = np.int64(rep.converged)
        times.update(vcycle_build_s=t_pinv, solve_s=t_solve)
        # one V-cycle apply on a fixed vector (operator-level parity)
        vin = np.random.default_rng(7).standard_normal(n)
        vin -= vin.mean()
        t3 = time.perf_counter()
        with threadpool_limits(1):
            vout = vop.apply(vin)
        times["vcycle_s"] = time.perf_counter() - t3
        vec_sig("vout", vout, store)
        print(f"{name}: its={rep.iterations} converged={rep.converged} solve {t_solve:.0f}s", flush=True)
    store["times_json"] = np.asarray(__import__("json").dumps(times))
    store["versions"] = np.asarray(f"numpy {np.__version__} scipy {__import__('scipy').__version__}")
    np.savez_compressed(OUT / f"big_{name}.npz", **store)
    print(f"{name}: written {times}", flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("names", nargs="+")
    ap.add_argument("--workers", type=int, default=6)
    a = ap.parse_args()
    for name in a.names:
        run(name, a.workers)


if __name__ == "__main__":
    main()
