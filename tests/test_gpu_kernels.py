"""GPU parity of the sparse kernels, the V-cycle and GMRES against the oracle.

Inputs are the reference's own golden fixtures; every comparison here is
bit-exact (SpMV / SpMM / Jacobi / transpose / residual) or within the stated
tolerance (coarsest GEMV inside the V-cycle, GMRES reductions).
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

from conftest import csr_from, gmres_args, oracle_cfg
from oracle import bamg_oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def eng():
    from paper_1402_4005_b200 import _lib, device
    _lib.lib()
    return _lib, device


def up(eng, M):
    return eng[1].DeviceCSR.from_host(M)


def dvec(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).cuda()


def test_spmv_bitexact(eng, golden):
    g = golden("kernels")
    A = csr_from(g, "A")
    dA = up(eng, A)
    y = torch.empty(A.shape[0], dtype=torch.float64, device="cuda")
    dx = dvec(g["x"])
    eng[0].call("bamg_spmv", dA.ref(), eng[0].ptr(dx), eng[0].ptr(y))
    assert np.array_equal(y.cpu().numpy(), g["Ax"])


def test_transpose_and_spmv_transpose_bitexact(eng, golden):
    g = golden("kernels")
    A = csr_from(g, "A")
    dA = up(eng, A)
    rp = torch.empty(A.shape[1] + 1, dtype=torch.int32, device="cuda")
    ci = torch.empty(A.nnz, dtype=torch.int32, device="cuda")
    va = torch.empty(A.nnz, dtype=torch.float64, device="cuda")
    eng[0].call("bamg_csr_transpose", dA.ref(), eng[0].ptr(rp), eng[0].ptr(ci), eng[0].ptr(va))
    ref = csr_from(g, "AT")
    assert np.array_equal(rp.cpu().numpy(), ref.indptr)
    assert np.array_equal(ci.cpu().numpy(), ref.indices)
    assert np.array_equal(va.cpu().numpy(), ref.data)
    dT = eng[1].DeviceCSR(rp, ci, va, (A.shape[1], A.shape[0]))
    y = torch.empty(A.shape[1], dtype=torch.float64, device="cuda")
    dx = dvec(g["x"])
    eng[0].call("bamg_spmv", dT.ref(), eng[0].ptr(dx), eng[0].ptr(y))
    assert np.array_equal(y.cpu().numpy(), g["ATx"])


@pytest.mark.parametrize("pair", [False, True])
@pytest.mark.parametrize("k", [1, 3, 8, 12, 16])
def test_spmm_bitexact(eng, k, pair, monkeypatch):
    if pair:
        monkeypatch.setenv("BAMG_PAIR_KERNEL", "1")
    rng = np.random.default_rng(k)
    from scipy import sparse as sp
    A = orc.canon(sp.random_array((3000, 2500), density=0.003, random_state=rng))
    X = rng.standard_normal((2500, k))
    dA = up(eng, A)
    Y = torch.empty((3000, k), dtype=torch.float64, device="cuda")
    dX = dvec(X)
    eng[0].call("bamg_spmm", dA.ref(), eng[0].ptr(dX), eng[0].ptr(Y), k)
    ref = np.stack([A @ X[:, c] for c in range(k)], axis=1)
    assert np.array_equal(Y.cpu().numpy(), ref)


def test_jacobi_bitexact_with_degenerate_rows(eng, golden):
    g = golden("kernels")
    B = csr_from(g, "jacB")
    d = B.diagonal()
    dB = up(eng, B)
    dd = dvec(d)
    skip = torch.empty(B.shape[0], dtype=torch.uint8, device="cuda")
    eng[0].call("bamg_degenerate_rows", dB.ref(), eng[0].ptr(dd), eng[0].ptr(skip))
    assert np.array_equal(skip.cpu().numpy().astype(bool), g["jac_skip"])
    out = torch.empty(B.shape[0], dtype=torch.float64, device="cuda")
    bb, xx = dvec(g["jac_b"]), dvec(g["jac_x"])  # keep the inputs alive across the call
    eng[0].call("bamg_jacobi", dB.ref(), eng[0].ptr(dd), eng[0].ptr(skip), eng[0].ptr(bb),
                None, eng[0].ptr(xx), eng[0].ptr(out), 1, 0.7, None)
    assert np.array_equal(out.cpu().numpy(), g["jac_out"])


def test_spgemm_identity_mass_flags_bitexact(eng):
    """(Q I) W == spgemm(Q, W, REV_A) and P^T (I P) == spgemm(P^T, P, REV_B), bit for bit."""
    import scipy.sparse as sp
    from paper_1402_4005_b200 import engine
    from paper_1402_4005_b200.device import DeviceCSR
    rng = np.random.default_rng(7)
    n, nc = 900, 240
    Q = sp.random(nc, n, density=0.02, random_state=rng, format="csr")
    Q.data = rng.standard_normal(Q.nnz)
    P = sp.random(n, nc, density=0.02, random_state=rng, format="csr")
    P.data = rng.standard_normal(P.nnz)
    Q.sort_indices()
    P.sort_indices()
    dQ, dW, dP = DeviceCSR.from_host(Q), DeviceCSR.from_host(Q.T.tocsr()), DeviceCSR.from_host(P)
    dPt = engine.transpose(dP)
    I = DeviceCSR.identity(n)
    a = engine.spgemm(engine.spgemm(dQ, I, order=1), dW, order=0).to_host()
    b = engine.spgemm(dQ, dW, order=engine.SPGEMM_REV_A).to_host()
    assert np.array_equal(a.indptr, b.indptr) and np.array_equal(a.indices, b.indices)
    assert np.array_equal(a.data.view(np.int64), b.data.view(np.int64))
    c = engine.spgemm(dPt, engine.spgemm(I, dP, order=1), order=0).to_host()
    d = engine.spgemm(dPt, dP, order=engine.SPGEMM_REV_B).to_host()
    assert np.array_equal(c.indptr, d.indptr) and np.array_equal(c.indices, d.indices)
    assert np.array_equal(c.data.view(np.int64), d.data.view(np.int64))


@pytest.mark.parametrize("mode", [0, 1, 2, 3])
def test_reciprocal_division_is_ieee_exact(eng, mode):
    """The Jacobi epilogue divides through RN(1/d) + one FMA correction; it must
    equal IEEE x / d bit for bit (2^28 random pairs per mode, 2 seeds)."""
    import ctypes as C
    for seed in (1, 12345):
        mis = C.c_int64(-1)
        eng[0].call("bamg_selftest_div", 1 << 28, seed, mode, C.byref(mis))
        assert mis.value == 0, f"mode {mode} seed {seed}: {mis.value} mismatches"


def _device_hierarchy(eng, levels, omega, nu1, nu2):
    """Upload an oracle-built hierarchy (test input) into an engine hierarchy."""
    import ctypes as C
    L = eng[0]
    keep = []
    h = C.c_void_p()
    L.check(L.lib().bamg_hier_create(L.ctx(), len(levels), C.byref(h)), "hier_create")
    for i, lv in enumerate(levels):
        dB = up(eng, lv.B)
        d = dvec(lv.d)
        sk = torch.from_numpy(orc.skip_rows(lv.B, lv.d).astype(np.uint8)).cuda()
        dP = up(eng, lv.P) if lv.P is not None else None
        dQ = up(eng, lv.Q) if lv.Q is not None else None
        keep += [dB, d, sk, dP, dQ]
        L.check(L.lib().bamg_hier_set_level(h, i, dB.ref(), L.ptr(d), L.ptr(sk),
                                            dP.ref() if dP else None, dQ.ref() if dQ else None), "set_level")
    A = levels[-1].B.toarray()
    U, s, Vt = np.linalg.svd(A)
    keep_s = s > 1e-12 * s[0]
    Z = (Vt[keep_s].T / s[keep_s]) @ U[:, keep_s].T
    dZ = dvec(np.ascontiguousarray(Z))
    keep.append(dZ)
    L.check(L.lib().bamg_hier_set_coarsest(h, L.ptr(dZ), A.shape[0]), "set_coarsest")
    L.check(L.lib().bamg_hier_set_smoother(h, omega, nu1, nu2), "set_smoother")
    return h, keep


@pytest.mark.parametrize("name", ["pipe_cfg0_tandem64", "pipe_planar1024_k12", "pipe_uniform63"])
@pytest.mark.parametrize("graphs", [True, False])
def test_vcycle_and_gmres_match_oracle(eng, golden, name, graphs, monkeypatch):
    import ctypes as C
    if not graphs:
        monkeypatch.setenv("BAMG_NO_GRAPHS", "1")
    g = golden(name)
    B = csr_from(g, "B")
    cfg = oracle_cfg(g)
    restart, max_iters, rtol = gmres_args(g)
    levels, T, x0 = orc.setup(B, cfg, g.get("geometry"), g["init_right_draw"], g["init_left_draw"])
    Cv = orc.VCycle(levels, cfg["omega"], cfg["nu_pre"], cfg["nu_post"])
    h, keep = _device_hierarchy(eng, levels, cfg["omega"], cfg["nu_pre"], cfg["nu_post"])
    L = eng[0]
    b = g["vcycle_in"]
    out = torch.empty(B.shape[0], dtype=torch.float64, device="cuda")
    db = dvec(b)
    L.call("bamg_vcycle", h, L.ptr(db), L.ptr(out))
    ref = Cv(b)
    got = out.cpu().numpy()
    assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max()
    assert np.abs(got - g["vcycle_out"]).max() <= 1e-12 * np.abs(ref).max()
    # GMRES
    dB = up(eng, B)
    x = torch.empty(B.shape[0], dtype=torch.float64, device="cuda")
    its = C.c_int(0)
    nh = C.c_int(0)
    hist = (C.c_double * (max_iters + 1))()
    zero, dx0 = torch.zeros_like(x), dvec(x0)
    rc = L.lib().bamg_gmres(L.ctx(), dB.ref(), h, L.ptr(zero), L.ptr(dx0), L.ptr(x),
                            -1 if restart is None else restart, max_iters, rtol, 0,
                            C.byref(its), hist, C.byref(nh))
    L.check(rc, "gmres")
    assert rc == 0
    assert its.value == int(g["iterations"])
    xs = orc.l1_sign_fix(x.cpu().numpy())
    assert np.abs(xs - g["x"]).sum() <= 1e-10
    L.lib().bamg_hier_destroy(h)


@pytest.mark.parametrize("name", ["pipe_cfg0_tandem64", "pipe_uniform63", "pipe_petri10_normal"])
def test_dense_pinv_bordered_lu_matches_svd(eng, golden, name, monkeypatch):
    """The bordered Gauss-Jordan pseudo-inverse (certified path) equals the
    reference's SVD pseudo-inverse of the coarsest operator; the forced SVD
    path (BAMG_PINV_SVD) agrees too."""
    from paper_1402_4005_b200 import engine
    g = golden(name)
    L = int(g["n_levels"]) - 1
    B = csr_from(g, f"L{L}_B")
    ref = np.linalg.pinv(B.toarray(), rcond=1e-12)
    dB = up(eng, B)
    D = engine.csr_to_dense(dB)
    for force in (False, True):
        if force:
            monkeypatch.setenv("BAMG_PINV_SVD", "1")
        Z = engine.dense_pinv(D, B.shape[0]).cpu().numpy()
        assert np.abs(Z - ref).max() <= 1e-9 * np.abs(ref).max(), force


@pytest.mark.parametrize("pool", [None, "64"])
@pytest.mark.parametrize("shape", [(300, 400, 500, 0.05, 0.03), (500, 500, 500, 0.004, 0.004),
                                   (400, 400, 600, 0.015, 0.013)])
def test_spgemm_matches_scipy_storage_order_and_canonical(eng, shape, pool, monkeypatch):
    """C = A B with scipy csr_matmat semantics: order 1 reproduces scipy's raw
    product arrays (reverse-first-touch rows) bit for bit, order 0 the
    canonical make_csr form.  The first shape has rows with > 64 distinct
    columns (global-scratch slow path), the second only shared-memory-tier
    rows (<= 32), the third all three tiers in one product (98 rows <= 32,
    237 with 33-64 through the local-memory tier, 65 > 64).
    pool = 64 starts the slow-path scratch pool at 64 entries, so the count
    overflows it, grows it and recounts."""
    from scipy import sparse as sp
    from paper_1402_4005_b200 import engine
    if pool:
        monkeypatch.setenv("BAMG_SPGEMM_POOL", pool)
    m, k, n, da, db = shape
    rng = np.random.default_rng(m + n)
    A = sp.random_array((m, k), density=da, format="csr", random_state=rng)
    B = sp.random_array((k, n), density=db, format="csr", random_state=rng)
    A = sp.csr_array(A)
    B = sp.csr_array(B)
    A.data = rng.standard_normal(A.nnz)
    B.data = rng.standard_normal(B.nnz)
    A.sort_indices()
    B.sort_indices()
    raw = A @ B  # scipy csr_matmat, unsorted rows
    dA, dB = up(eng, A), up(eng, B)
    C1 = engine.spgemm(dA, dB, order=1).to_host()
    assert np.array_equal(C1.indptr, raw.indptr)
    assert np.array_equal(C1.indices, raw.indices)
    assert np.array_equal(C1.data, raw.data)
    C0 = engine.spgemm(dA, dB, order=0).to_host()
    ref = orc.canon(raw)
    assert np.array_equal(C0.indptr, ref.indptr) and np.array_equal(C0.indices, ref.indices)
    assert np.array_equal(C0.data, ref.data)


@pytest.mark.parametrize("kind", ["lattice", "lattice_sparse", "negative", "fractional", "signed_zero"])
def test_axis_ranks_match_numpy_unique_inverse(eng, kind):
    """Per-axis ranks among the distinct coordinate values (np.unique's inverse,
    coarsen.py:90-109): the integer presence/scan fast path (lattice
    coordinates) and the 64-bit radix path (everything else) agree with numpy."""
    from paper_1402_4005_b200 import engine
    rng = np.random.default_rng(7)
    n = 50_000
    if kind == "lattice":
        x = rng.integers(0, 1024, n).astype(np.float64)
    elif kind == "lattice_sparse":
        x = (rng.integers(0, 300, n) * 37).astype(np.float64)
    elif kind == "negative":
        x = rng.integers(-500, 500, n).astype(np.float64)
    elif kind == "fractional":
        x = np.round(rng.random(n) * 1000, 3)
    else:
        x = rng.integers(0, 3, n).astype(np.float64) - 1.0
        x[x == 0] = -0.0
        x[::7] = 0.0
    rank, nv = engine.axis_ranks(dvec(x))
    vals, inv = np.unique(x, return_inverse=True)
    assert nv == len(vals)
    assert np.array_equal(rank.cpu().numpy(), inv.astype(np.int32))


def test_spgemm_many_matches_single_products(eng):
    """Independent products counted together (one host read) give exactly the
    arrays of the one-at-a-time products, in every order mode."""
    from scipy import sparse as sp
    from paper_1402_4005_b200 import engine
    rng = np.random.default_rng(3)
    mats = []
    for (m, k, n, d) in [(300, 400, 350, 0.02), (200, 300, 250, 0.05), (120, 120, 120, 0.2)]:
        A = sp.csr_array(sp.random_array((m, k), density=d, format="csr", random_state=rng))
        B = sp.csr_array(sp.random_array((k, n), density=d, format="csr", random_state=rng))
        A.data = rng.standard_normal(A.nnz)
        B.data = rng.standard_normal(B.nnz)
        A.sort_indices()
        B.sort_indices()
        mats.append((up(eng, A), up(eng, B)))
    prods = [(mats[0][0], mats[0][1], 1), (mats[1][0], mats[1][1], engine.SPGEMM_REV_A),
             (mats[2][0], mats[2][1], engine.SPGEMM_REV_B | 1)]
    many = engine.spgemm_many(prods)
    for (A, B, order), C in zip(prods, many):
        ref = engine.spgemm(A, B, order=order).to_host()
        got = C.to_host()
        assert np.array_equal(got.indptr, ref.indptr) and np.array_equal(got.indices, ref.indices)
        assert np.array_equal(got.data, ref.data)


@pytest.mark.parametrize("family,side", [("tandem", 2), ("tandem", 17), ("tandem", 64), ("uniform2d", 2),
                                         ("uniform2d", 33), ("uniform2d", 128)])
def test_device_lattice_chain_matches_host(eng, family, side):
    """On-device assembly of B: the same canonical CSR
    arrays and geometry as the host generators, bit for bit."""
    from paper_1402_4005_b200 import chains
    host = chains.tandem_queue(side) if family == "tandem" else chains.uniform_2d(side)
    dev = chains.lattice_chain_device(family, side)
    H = host.B
    D = dev.B.to_host()
    assert np.array_equal(D.indptr, H.indptr) and np.array_equal(D.indices, H.indices)
    assert np.array_equal(D.data, H.data)
    assert np.array_equal(dev.geometry.cpu().numpy().T, host.geometry)


@pytest.mark.parametrize("seed,k,n", [(0, 8, 1), (0, 16, 1000), (0, 8, 100_003), (7, 12, 4097)])
def test_device_uniform_draws_match_numpy(eng, seed, k, n):
    """BASELINE's test vectors drawn on the device (numpy PCG64 jump-ahead):
    default_rng(seed).random((k, n)) twice, bit for bit, n x k interleaved."""
    from paper_1402_4005_b200 import engine
    g = np.random.default_rng(seed)
    right, left = g.random((k, n)), g.random((k, n))
    dr, dl = engine.uniform_draws(seed, k, n)
    assert np.array_equal(dr.cpu().numpy(), right.T) and np.array_equal(dl.cpu().numpy(), left.T)


@pytest.mark.parametrize("n", [4, 5, 100, 1024, 30_000])
def test_device_planar_chain_matches_host(eng, n):
    """On-device assembly of the planar chain from its Delaunay triangles
    (remainder): the host generator's canonical CSR of
    B = I - A and the point geometry, bit for bit."""
    from paper_1402_4005_b200 import chains
    host = chains.random_planar(n, seed=1)
    dev = chains.planar_chain_device(n, seed=1)
    H = host.B
    D = dev.B.to_host()
    assert np.array_equal(D.indptr, H.indptr) and np.array_equal(D.indices, H.indices)
    assert np.array_equal(D.data, H.data)
    assert np.array_equal(dev.geometry.cpu().numpy().T, host.geometry)


@pytest.mark.gpu
@pytest.mark.parametrize("k", [1, 3, 8, 16])
def test_block_kernels_match_numpy(eng, k):
    """n x k block kernels (flat double2 forms for k = 8, 16; row forms
    otherwise): column division is the IEEE quotient bit for bit (exact
    reciprocal path), row gathers and column permutations are copies, column
    norms agree with numpy to rounding (fixed-tree sums, not numpy's pairwise
    order)."""
    import torch
    from paper_1402_4005_b200 import engine
    rng = np.random.default_rng(11 + k)
    n = 40_003
    X = rng.standard_normal((n, k)) * np.exp(rng.uniform(-30, 30, (1, k)))
    dX = torch.from_numpy(X.copy()).cuda()
    nrm = engine.col_norms(dX).cpu().numpy()
    ref = np.sqrt((X * X).sum(axis=0))
    assert np.allclose(nrm, ref, rtol=1e-13, atol=0)
    engine.normalize_cols(dX)
    assert np.array_equal(dX.cpu().numpy(), X / nrm[None, :])
    idx = rng.integers(0, n, 9_001).astype(np.int32)
    G = engine.gather_rows(torch.from_numpy(X).cuda(), torch.from_numpy(idx).cuda()).cpu().numpy()
    assert np.array_equal(G, X[idx])
    perm = rng.permutation(k).astype(np.int32)
    Pm = engine.permute_cols(torch.from_numpy(X).cuda(), perm).cpu().numpy()
    assert np.array_equal(Pm, X[:, perm])


@pytest.mark.parametrize("family,side", [("tandem", 63), ("uniform2d", 40), ("planar", 1500),
                                         ("tandem", 700), ("uniform2d", 611)])
def test_packed_operator_kernels_bitexact(eng, family, side):
    """bamg_csr_pack: the k = 1 SpMV / residual / Jacobi kernels on the packed
    (value-indexed, 32-bit) copy of a generator chain's B reproduce the CSR
    kernels -- and scipy's csr_matvec -- bit for bit (sparse.py:81-86, relax.py:66-83)."""
    from paper_1402_4005_b200 import chains, engine
    if family == "planar":
        prob = chains.random_planar(side, seed=1)
    elif family == "tandem":
        prob = chains.tandem_queue(side)
    else:
        prob = chains.uniform_2d(side)
    B = orc.canon(prob.B)
    n = B.shape[0]
    dB = up(eng, B)
    plain = up(eng, B)
    assert engine.pack_operator(dB)
    assert dB.packed is not None and dB.desc().packed
    # stencil tiles (bamg_csr_pack_stencil): the big lattices sweep most 256-row tiles from the
    # interior row's entry list, the small ones (every tile crosses a lattice line) and the mesh do not
    if family != "planar" and side >= 600:
        assert dB.ptiles is not None and dB.desc().ptiles
        assert 0.5 < float(dB.ptiles.sum()) / dB.ptiles.numel() < 1.0
        assert dB.desc().st_w == int(np.diff(B.indptr)[n // 2 + side // 4])
    else:
        assert dB.ptiles is None and not dB.desc().ptiles
    rng = np.random.default_rng(7)
    x, b = rng.standard_normal(n), rng.standard_normal(n)
    dx, db = dvec(x), dvec(b)
    # SpMV
    y = engine.spmm(dB, dx)
    assert np.array_equal(y.cpu().numpy(), B @ x)
    assert torch.equal(y, engine.spmm(plain, dx))
    # residual
    r = torch.empty_like(dx)
    r0 = torch.empty_like(dx)
    eng[0].call("bamg_residual", dB.ref(), eng[0].ptr(db), eng[0].ptr(dx), eng[0].ptr(r))
    eng[0].call("bamg_residual", plain.ref(), eng[0].ptr(db), eng[0].ptr(dx), eng[0].ptr(r0))
    assert torch.equal(r, r0)
    assert np.array_equal(r.cpu().numpy(), b - B @ x)
    # Jacobi (homogeneous and with a right-hand side), against the CSR kernel and the oracle
    d = engine.diag(plain)
    skip = engine.degenerate_rows(plain, d)
    for rhs in (None, db):
        got = engine.jacobi(dB, d, skip, dx, b=rhs)
        assert torch.equal(got, engine.jacobi(plain, d, skip, dx, b=rhs))
        dg = B.diagonal()
        want = orc.sweep(B, x, np.zeros(n) if rhs is None else b, 0.7, dg, orc.skip_rows(B, dg))
        assert np.array_equal(got.cpu().numpy(), want)

@pytest.mark.parametrize("family,side,k", [("tandem", 700, 16), ("uniform2d", 611, 8), ("tandem", 900, 8)])
def test_stencil_tiles_wide_sweeps_bitexact(eng, family, side, k):
    """bamg_csr_stencil: the k-wide SpMM / Jacobi sweeps (right-hand side, per-vector scale, peak)
    and the fused Rayleigh quotients of a lattice operator and of its transpose, taken from the
    stencil tiles, reproduce the CSR row kernels bit for bit (relax.py:66-83, bootstrap.py:144-153)."""
    from paper_1402_4005_b200 import chains, engine
    prob = chains.tandem_queue(side) if family == "tandem" else chains.uniform_2d(side)
    B = orc.canon(prob.B)
    n = B.shape[0]
    for M in (B, orc.canon(B.T)):
        dS, dP = up(eng, M), up(eng, M)
        assert engine.attach_stencil(dS) and dS.desc().ptiles and dS.desc().st_w >= 3
        rng = np.random.default_rng(11)
        X = torch.from_numpy(rng.standard_normal((n, k))).cuda()
        Bv = torch.from_numpy(rng.standard_normal((n, k))).cuda()
        sc = torch.from_numpy(rng.uniform(0.5, 2.0, k)).cuda()
        assert torch.equal(engine.spmm(dS, X), engine.spmm(dP, X))
        assert np.array_equal(engine.spmm(dS, X).cpu().numpy(), M @ X.cpu().numpy())
        d = engine.diag(dP)
        skip = engine.degenerate_rows(dP, d)
        for rhs, scale in ((None, None), (Bv, None), (Bv, sc)):
            pk_s = torch.zeros(k, dtype=torch.float64, device="cuda")
            pk_p = torch.zeros(k, dtype=torch.float64, device="cuda")
            got = engine.jacobi(dS, d, skip, X, b=rhs, b_scale=scale, peak=pk_s)
            want = engine.jacobi(dP, d, skip, X, b=rhs, b_scale=scale, peak=pk_p)
            assert torch.equal(got, want)
            assert torch.equal(pk_s, pk_p)
            assert torch.equal(engine.jacobi(dS, d, skip, X, b=rhs, b_scale=scale),
                               engine.jacobi(dP, d, skip, X, b=rhs, b_scale=scale))
        # Rayleigh quotients u.(Av) / (|u| |v|) with identity masses: same partial-sum tree
        U = torch.from_numpy(rng.standard_normal((n, k))).cuda()
        sig_s = torch.ones(k, dtype=torch.float64, device="cuda")
        sig_p = torch.ones(k, dtype=torch.float64, device="cuda")
        engine.refresh_sigmas(dS, None, None, U, X, sig_s, flip=False)
        engine.refresh_sigmas(dP, None, None, U, X, sig_p, flip=False)
        assert torch.equal(sig_s, sig_p)


def test_pack_operator_declines_general_values(eng):
    """More than 256 distinct values (any Galerkin operator): not packed, CSR kernels run."""
    from scipy import sparse as sp
    from paper_1402_4005_b200 import engine
    rng = np.random.default_rng(3)
    A = orc.canon(sp.random_array((2000, 2000), density=0.004, random_state=rng) + sp.eye_array(2000))
    dA = up(eng, A)
    assert not engine.pack_operator(dA)
    assert dA.packed is None and not dA.desc().packed
    x = rng.standard_normal(2000)
    assert np.array_equal(engine.spmm(dA, dvec(x)).cpu().numpy(), A @ x)
