"""Generate the golden fixtures under tests/golden/ by running the REFERENCE.

This script is the only place that imports the upstream reference package
(`markovmg`, read-only at /root/reference/pkg/src).  It runs in the build
container only; the fixtures it writes (`*.npz`) are committed and are what
the tests, `smoke()` and the oracle pins read on any machine.

Usage:  OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden.py [case ...]

Every case records the reference's own outputs for one seeded input:
  * pipeline cases (`pipe_*`): the whole `run_setup` + `gmres` path
    (bootstrap.py:395-429, solver.py:136-226) with per-level C/F splits,
    P / Q / B_l / M_l / N_l in CSR form, the singular-test weights, the
    triplets after every smoothing block, x0, x, the iteration count and the
    residual history;
  * kernel cases (`kern_*`): spmv / spmv_transpose / transpose /
    triple_product / adjacency_structure (sparse.py), weighted Jacobi with
    degenerate rows (relax.py), fit_row (interp.py:129-238), cr_coarsen
    (coarsen.py:112-169), coarsest_triplets (bootstrap.py:205-281) and
    PinvOperator (dense.py:118-131) on small seeded inputs.
"""

from __future__ import annotations

import sys
import time
from pathlib import Path

import numpy as np
from scipy import sparse as sp

REF = "/root/reference/pkg/src"
OUT = Path(__file__).resolve().parent

sys.path.insert(0, REF)
from markovmg import bootstrap, chains, coarsen, dense, interp, presets, relax, solver  # noqa: E402
from markovmg import sparse as msparse  # noqa: E402


def csr_pack(prefix, M, store):
    M = sp.csr_array(M)
    store[prefix + "_indptr"] = np.asarray(M.indptr, dtype=np.int64)
    store[prefix + "_indices"] = np.asarray(M.indices, dtype=np.int64)
    store[prefix + "_data"] = np.asarray(M.data, dtype=np.float64)
    store[prefix + "_shape"] = np.asarray(M.shape, dtype=np.int64)


class UniformShim:
    """rng stand-in: `.standard_normal(shape)` returns the BASELINE uniform draws.

    BASELINE.json asks for k uniform(0,1) test vectors with seed 0; the
    reference draws standard normals (bootstrap.py:187-188).  Both paths take
    `default_rng(seed).random((k, n))` twice (right, then left).
    """

    def __init__(self, seed, k, n):
        g = np.random.default_rng(seed)
        self.draws = [g.random((k, n)), g.random((k, n))]
        self.calls = 0

    def standard_normal(self, shape):
        out = self.draws[self.calls]
        assert out.shape == tuple(shape)
        self.calls += 1
        return out.copy()


def run_pipeline(name, problem, cfg, gcfg, init_seed=None):
    """Run the reference on one problem and record every per-level artifact."""
    store = {}
    rec = {"splits": [], "P": [], "Q": [], "Bc": [], "vw": [], "uw": [], "smooth": []}

    orig_split = bootstrap.make_splitting
    orig_stw = bootstrap.singular_test_weights
    orig_bi = bootstrap.build_interpolation
    orig_br = bootstrap.build_restriction
    orig_sb = bootstrap._smooth_block
    orig_init = bootstrap.init_test_vectors

    def rec_split(B, geometry, ccfg, seed=None):
        s = orig_split(B, geometry, ccfg, seed)
        rec["splits"].append(s.coarse.copy())
        return s

    def rec_stw(B, vectors, transpose_side=False, infinite_slot=None):
        t = orig_stw(B, vectors, transpose_side, infinite_slot)
        rec["uw" if transpose_side else "vw"].append(t.weights.copy())
        return t

    def rec_bi(*a, **k):
        P = orig_bi(*a, **k)
        rec["P"].append(P)
        return P

    def rec_br(*a, **k):
        Q = orig_br(*a, **k)
        rec["Q"].append(Q)
        return Q

    def rec_sb(B, diag, M, N, trips, cfg_, inhomogeneous):
        orig_sb(B, diag, M, N, trips, cfg_, inhomogeneous)
        rec["smooth"].append((B.shape[0], bool(inhomogeneous), trips.sigmas.copy(),
                              trips.left.copy(), trips.right.copy()))

    init_vectors = {}

    def rec_init(B, cfg_, rng=None):
        if init_seed is not None:
            rng = UniformShim(init_seed, cfg_.n_tests, B.shape[0])
            init_vectors["right"] = rng.draws[0].copy()
            init_vectors["left"] = rng.draws[1].copy()
        else:
            # record the standard-normal draws the reference makes itself
            state = rng.bit_generator.state
            init_vectors["right"] = rng.standard_normal((cfg_.n_tests, B.shape[0]))
            init_vectors["left"] = rng.standard_normal((cfg_.n_tests, B.shape[0]))
            rng.bit_generator.state = state
        t = orig_init(B, cfg_, rng)
        store["init_sigmas"] = t.sigmas.copy()
        store["init_left"] = t.left.copy()
        store["init_right"] = t.right.copy()
        return t

    bootstrap.make_splitting = rec_split
    bootstrap.singular_test_weights = rec_stw
    bootstrap.build_interpolation = rec_bi
    bootstrap.build_restriction = rec_br
    bootstrap._smooth_block = rec_sb
    bootstrap.init_test_vectors = rec_init
    try:
        t0 = time.perf_counter()
        setup = bootstrap.run_setup(problem, cfg)
        t1 = time.perf_counter()
        vop = solver.VCycleOperator(setup.hierarchy, cfg.smoother)
        rep = solver.gmres(problem.B, np.zeros(problem.n), setup.x0, gcfg, precond=vop)
        t2 = time.perf_counter()
        # one V-cycle apply on a fixed vector, for operator-level parity
        vin = np.random.default_rng(7).standard_normal(problem.n)
        vin -= vin.mean()
        vout = vop.apply(vin)
    finally:
        bootstrap.make_splitting = orig_split
        bootstrap.singular_test_weights = orig_stw
        bootstrap.build_interpolation = orig_bi
        bootstrap.build_restriction = orig_br
        bootstrap._smooth_block = orig_sb
        bootstrap.init_test_vectors = orig_init

    csr_pack("B", problem.B, store)
    if problem.geometry is not None:
        store["geometry"] = problem.geometry
    store["init_right_draw"] = init_vectors["right"]
    store["init_left_draw"] = init_vectors["left"]
    h = setup.hierarchy
    store["n_levels"] = np.int64(h.depth)
    for li, lev in enumerate(h.levels):
        csr_pack(f"L{li}_B", lev.B, store)
        csr_pack(f"L{li}_M", lev.M, store)
        csr_pack(f"L{li}_N", lev.N, store)
        if lev.P is not None:
            csr_pack(f"L{li}_P", lev.P, store)
            csr_pack(f"L{li}_Q", lev.Q, store)
            store[f"L{li}_coarse"] = lev.split.coarse
    # every split attempted (including a truncated last one) and every fit
    for i, c in enumerate(rec["splits"]):
        store[f"split{i}"] = c
    store["n_splits"] = np.int64(len(rec["splits"]))
    for i, w in enumerate(rec["vw"]):
        store[f"vw{i}"] = w
    for i, w in enumerate(rec["uw"]):
        store[f"uw{i}"] = w
    store["n_fits"] = np.int64(len(rec["vw"]))
    for i, P in enumerate(rec["P"]):
        csr_pack(f"fitP{i}", P, store)
    for i, Q in enumerate(rec["Q"]):
        csr_pack(f"fitQ{i}", Q, store)
    for i, (n, inh, s, lft, rgt) in enumerate(rec["smooth"]):
        store[f"sm{i}_meta"] = np.asarray([n, int(inh)], dtype=np.int64)
        store[f"sm{i}_sigmas"] = s
        store[f"sm{i}_left"] = lft
        store[f"sm{i}_right"] = rgt
    store["n_smooth"] = np.int64(len(rec["smooth"]))
    store["trip_sigmas"] = setup.triplets.sigmas
    store["trip_left"] = setup.triplets.left
    store["trip_right"] = setup.triplets.right
    store["x0"] = setup.x0
    store["x"] = solver._sign_fix_l1(rep.x)
    store["x_raw"] = rep.x
    store["iterations"] = np.int64(rep.iterations)
    store["history"] = np.asarray(rep.residual_history)
    store["converged"] = np.int64(rep.converged)
    store["vcycle_in"] = vin
    store["vcycle_out"] = vout
    o_g, o_c, depth = bootstrap.complexities(h)
    store["complexities"] = np.asarray([o_g, o_c, depth])
    # configuration, so the consumer can rebuild the identical config
    store["cfg_ints"] = np.asarray([cfg.n_tests, cfg.setup_cycles, cfg.inner_passes,
                                    cfg.smoother.sweeps_pre, cfg.smoother.sweeps_post,
                                    cfg.interp.caliber, cfg.interp.search_radius,
                                    int(cfg.interp.constrain_constant_in_q),
                                    int(cfg.interp.nonnegative),
                                    cfg.coarsening.stop_size, cfg.coarsening.cr_sweeps,
                                    cfg.coarsening.max_levels, cfg.seed,
                                    -1 if init_seed is None else init_seed], dtype=np.int64)
    store["cfg_floats"] = np.asarray([cfg.smoother.omega, cfg.interp.improvement_tol,
                                      cfg.coarsening.cr_threshold, cfg.coarsening.cr_omega],
                                     dtype=np.float64)
    store["cfg_mode"] = np.asarray(cfg.coarsening.mode)
    store["family"] = np.asarray(problem.family)
    store["gmres"] = np.asarray([-1 if gcfg.restart is None else gcfg.restart,
                                 gcfg.max_iters, gcfg.rtol], dtype=np.float64)
    store["ref_seconds"] = np.asarray([t1 - t0, t2 - t1])
    np.savez_compressed(OUT / f"{name}.npz", **store)
    print(f"{name}: n={problem.n} levels={h.depth} its={rep.iterations} "
          f"setup={t1 - t0:.2f}s solve={t2 - t1:.3f}s")


def pipeline_cases():
    cases = {}

    def tandem(side, k, stop, restart=None, rtol=1e-8, seed_init=0):
        prob = chains.tandem_queue(side)
        cfg = presets.default_setup_config("tandem", cycles=1, seed=0, n_tests=k)
        cfg = _with_stop(cfg, stop)
        return prob, cfg, solver.GmresConfig(restart=restart, rtol=rtol), seed_init

    # cfg0 of BASELINE.json exactly: tandem 64x64, k=8, coarsest <= 64
    cases["pipe_cfg0_tandem64"] = lambda: tandem(64, 8, 65)
    # cfg2 shape at desk scale: k = 16, restart 30
    cases["pipe_tandem32_k16_r30"] = lambda: tandem(32, 16, 290, restart=30)

    def uniform(side, k=8):
        prob = chains.uniform_2d(side)
        cfg = presets.default_setup_config("uniform2d", cycles=1, seed=0, n_tests=k)
        return prob, cfg, solver.GmresConfig(rtol=1e-8), 0

    cases["pipe_uniform33"] = lambda: uniform(33)
    cases["pipe_uniform63"] = lambda: uniform(63)

    def two_cycles(fam, side, k):
        prob = chains.tandem_queue(side) if fam == "tandem" else chains.uniform_2d(side)
        cfg = presets.default_setup_config(fam, cycles=2, seed=0, n_tests=k)
        return prob, cfg, solver.GmresConfig(rtol=1e-8), 0

    # BAMG^2: a second setup cycle with inhomogeneous smoothing on every level
    cases["pipe2_tandem33_bamg2"] = lambda: two_cycles("tandem", 33, 8)
    cases["pipe2_uniform33_bamg2"] = lambda: two_cycles("uniform2d", 33, 8)

    def planar(n, k=12):
        prob = chains.random_planar(n, seed=1)
        cfg = presets.default_setup_config("planar", cycles=1, seed=0, n_tests=k)
        return prob, cfg, solver.GmresConfig(rtol=1e-8), 0

    cases["pipe_planar1024_k12"] = lambda: planar(1024)

    def bd(n):
        prob = chains.birth_death(n)
        cfg = presets.default_setup_config("birth-death", cycles=1, seed=1)
        return prob, cfg, solver.GmresConfig(rtol=1e-7), None

    # reference's own standard-normal init (no shim), seed 1, 1-D geometric
    cases["pipe_bd257_normal"] = lambda: bd(257)

    def petri(tokens):
        prob = presets.build_problem("petri", tokens=tokens)
        cfg = presets.default_setup_config("petri", cycles=1, seed=1)
        return prob, cfg, solver.GmresConfig(rtol=1e-7), None

    # Petri: fine points with no coarse point within two hops (empty rows)
    cases["pipe_petri10_normal"] = lambda: petri(10)
    return cases


def _with_stop(cfg, stop):
    from dataclasses import replace
    return replace(cfg, coarsening=replace(cfg.coarsening, stop_size=stop))


def kernel_cases():
    store = {}
    rng = np.random.default_rng(2024)
    # --- sparse.py: random nonsymmetric CSR with an empty row and mixed signs
    n = 300
    A = sp.random_array((n, n), density=0.02, format="csr", random_state=rng)
    A = sp.csr_array(A)
    A.data = rng.standard_normal(A.nnz)
    A = A.tolil()
    A[5, :] = 0.0
    A = msparse.make_csr(A)
    x = rng.standard_normal(n)
    csr_pack("A", A, store)
    store["x"] = x
    store["Ax"] = msparse.spmv(A, x)
    store["ATx"] = msparse.spmv_transpose(A, x)
    csr_pack("AT", msparse.transpose(A), store)
    csr_pack("adjA", msparse.adjacency_structure(A), store)
    # triple product on a chain with LS transfer operators of the reference
    prob = chains.uniform_2d(17)
    cfg = presets.default_setup_config("uniform2d", seed=1)
    split = coarsen.geometric_coarsen(prob.geometry, "geometric2d")
    trips = bootstrap.init_test_vectors(prob.B, cfg, np.random.default_rng(5))
    vt = interp.singular_test_weights(prob.B, trips.right)
    ut = interp.singular_test_weights(prob.B, trips.left, True, 0)
    P = interp.build_interpolation(prob.B, split, vt, cfg.interp)
    Q = interp.build_restriction(prob.B, split, ut, cfg.interp)
    csr_pack("tpB", prob.B, store)
    csr_pack("tpP", P, store)
    csr_pack("tpQ", Q, store)
    csr_pack("tpC", msparse.triple_product(Q, prob.B, P), store)
    store["tp_coarse"] = split.coarse
    store["tp_right"] = trips.right
    store["tp_left"] = trips.left
    store["tp_vw"] = vt.weights
    store["tp_uw"] = ut.weights
    # --- relax.py: weighted Jacobi with degenerate rows (nonpositive / dominated)
    Bj = prob.B.tolil()
    Bj[3, 3] = 0.0
    Bj[7, 7] = -0.5
    Bj[11, 11] = 0.01
    Bj = msparse.make_csr(Bj)
    sm = relax.SmootherConfig()
    xb = rng.standard_normal(prob.n)
    bb = rng.standard_normal(prob.n)
    d = Bj.diagonal()
    store["jac_skip"] = relax.degenerate_rows(Bj, d)
    store["jac_skip_t"] = relax.degenerate_rows(Bj, d, transpose=True)
    csr_pack("jacB", Bj, store)
    store["jac_x"] = xb
    store["jac_b"] = bb
    store["jac_out"] = relax.jacobi_sweep(Bj, xb, bb, sm, d)
    store["jac_out_t"] = relax.jacobi_sweep_transpose(Bj, xb, bb, sm, d)
    # --- interp.py: fit_row on seeded small problems, every flag combination
    fits = []
    for t in range(64):
        r = int(rng.integers(2, 17))
        m = int(rng.integers(1, 10))
        y = rng.random(r) if t % 3 else rng.standard_normal(r)
        C = rng.random((r, m)) if t % 2 else rng.standard_normal((r, m))
        w = rng.random(r) * 10.0 + 1e-3
        if t % 4 == 0:
            w[0] = np.inf
        cal = int(rng.integers(1, 5))
        constrain = bool(t % 4 == 0 or t % 5 == 0)
        nonneg = bool(t % 7 != 3)
        ridge = float(rng.choice([0.0, 0.01, 0.3]))
        sel, coef, val = interp.fit_row(y, C, w, cal, 1e-3, constrain=constrain,
                                        ridge=ridge, nonnegative=nonneg)
        fits.append((r, m, cal, int(constrain), int(nonneg), ridge, y, C, w, sel, coef, val))
    store["fit_n"] = np.int64(len(fits))
    for i, (r, m, cal, con, nn, ridge, y, C, w, sel, coef, val) in enumerate(fits):
        store[f"fit{i}_meta"] = np.asarray([r, m, cal, con, nn], dtype=np.int64)
        store[f"fit{i}_ridge"] = np.float64(ridge)
        store[f"fit{i}_y"] = y
        store[f"fit{i}_C"] = C
        store[f"fit{i}_w"] = w
        store[f"fit{i}_sel"] = sel
        store[f"fit{i}_coef"] = coef
        store[f"fit{i}_val"] = np.float64(val)
    # --- coarsen.py: CR on a small planar chain
    pl = chains.random_planar(400, seed=3)
    ccfg = coarsen.CoarseningConfig(mode="cr", cr_threshold=0.78)
    ss = np.random.SeedSequence(11)
    csr_pack("crB", pl.B, store)
    store["cr_coarse"] = coarsen.cr_coarsen(pl.B, ccfg, ss).coarse
    # --- bootstrap.py: coarsest triplets on a small Galerkin-like level
    small = chains.tandem_queue(8)
    Md = sp.csr_array(np.diag(rng.random(small.n) + 0.5))
    Nd = sp.csr_array(np.diag(rng.random(small.n) + 0.5))
    tr = bootstrap.coarsest_triplets(small.B, Md, Nd, 6)
    csr_pack("ctB", small.B, store)
    store["ct_M"] = Md.diagonal()
    store["ct_N"] = Nd.diagonal()
    store["ct_sigmas"] = tr.sigmas
    store["ct_left"] = tr.left
    store["ct_right"] = tr.right
    # --- dense.py: pseudoinverse of a singular chain operator
    pin = dense.PinvOperator(small.B.toarray())
    bvec = rng.standard_normal(small.n)
    store["pinv_b"] = bvec
    store["pinv_out"] = pin.apply(bvec)
    np.savez_compressed(OUT / "kernels.npz", **store)
    print("kernels: written")


def main(argv):
    cases = pipeline_cases()
    names = argv or (list(cases) + ["kernels"])
    for name in names:
        if name == "kernels":
            kernel_cases()
            continue
        prob, cfg, gcfg, seed_init = cases[name]()
        run_pipeline(name, prob, cfg, gcfg, init_seed=seed_init)


if __name__ == "__main__":
    main(sys.argv[1:])
