"""Full-size parity checks against the reference-generated `big_cfgX.npz` fixtures.

The fixtures (tests/golden/make_golden_big.py, which ran the unmodified
reference on BASELINE.json configs 1-4) hold compact signatures: sha256 of
every split and of every operator's indptr / indices, value checksums, the
GMRES iteration count and x (full for cfg1/cfg2; every 64th entry and 4,096
block sums for cfg4).  `check_config` runs the GPU path on the same seeded
inputs and compares.  Used by tests/test_gpu_big.py and, after its timed
region, by bench.py's `parity` field (checker only; never on a timed path).
"""

from __future__ import annotations

import hashlib
from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"


def fixture(name):
    p = GOLDEN / f"big_{name}.npz"
    if not p.exists():
        return None
    with np.load(p, allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(np.asarray(a, dtype=np.int64)).tobytes()).hexdigest()


def _host_csr(M, n=None):
    """(indptr, indices, data) of a DeviceCSR, a scipy matrix, or None (= identity of size n)."""
    if M is None:
        return np.arange(n + 1), np.arange(n), np.ones(n)
    if hasattr(M, "rowptr"):
        return (M.rowptr.cpu().numpy(), M.col.cpu().numpy(), M.val.cpu().numpy())
    return M.indptr, M.indices, M.data


def csr_mismatch(g, prefix, M, n=None, rel=1e-9):
    """None if the operator matches the fixture signature, else a message."""
    ip, ix, v = _host_csr(M, n)
    if int(g[prefix + "_nnz"]) != ix.size:
        return f"{prefix}: nnz {ix.size} != {int(g[prefix + '_nnz'])}"
    if sha(ip) != str(g[prefix + "_sha_indptr"]) or sha(ix) != str(g[prefix + "_sha_indices"]):
        return f"{prefix}: sparsity pattern differs"
    ref = g[prefix + "_vsum"]
    proj = np.random.default_rng(12345).standard_normal(v.size) @ v
    scale = max(float(ref[1]), 1e-300)
    if abs(np.abs(v).sum() - ref[1]) > rel * scale or abs(v.sum() - ref[0]) > rel * scale \
            or abs(proj - ref[2]) > 5 * rel * scale:
        return f"{prefix}: values differ (sum {v.sum():.17g} vs {ref[0]:.17g})"
    return None


def vec_errors(g, prefix, x):
    """(estimated l1 error from the every-64th sample, block-sum l1 lower bound, full l1 or None)."""
    x = np.asarray(x, dtype=np.float64)
    est = 64.0 * float(np.abs(x[::64] - g[prefix + "_every64"]).sum())
    blocks = np.add.reduceat(x, np.linspace(0, x.size, 4097).astype(np.int64)[:-1])
    low = float(np.abs(blocks - g[prefix + "_blocks"]).sum())
    full = float(np.abs(x - g[prefix]).sum()) if prefix in g else None
    return est, low, full


def run_config(name, setup_only=False):
    """Run our path on a BASELINE config with the fixture's inputs; returns (problem, cfg, setup, reports)."""
    import torch

    import bench
    import paper_1402_4005_b200 as pb
    from paper_1402_4005_b200.chains import ChainProblem
    from paper_1402_4005_b200.device import DeviceCSR

    fam, size, k, stop, restart, _ = bench.CONFIGS[name]
    prob = bench.build_problem(name)
    cfg = bench.setup_config(name)
    right, left = bench.draws_for(k, prob.n)
    dB = DeviceCSR.from_host(prob.B)
    dV = torch.from_numpy(np.ascontiguousarray(right.T)).cuda()
    dU = torch.from_numpy(np.ascontiguousarray(left.T)).cuda()
    geo = torch.from_numpy(np.ascontiguousarray(prob.geometry.T)).cuda()
    dprob = ChainProblem(A=None, B=dB, n=prob.n, family=fam, params={}, geometry=geo)
    setup = pb.run_setup(dprob, cfg, draws=(dV, dU), B_device=dB)
    return prob, dB, cfg, setup


def check_config(name, g=None, result=None):
    """Compare one config with its fixture.  Returns a dict of findings
    (`ok`, `failures`, iteration counts, x errors)."""
    import torch

    import bench
    import paper_1402_4005_b200 as pb
    from paper_1402_4005_b200.solver import _sign_fix_l1

    g = g if g is not None else fixture(name)
    if g is None:
        return {"ok": None, "why": f"no fixture big_{name}.npz"}
    prob, dB, cfg, setup = result if result is not None else run_config(name)
    fails = []
    m = csr_mismatch(g, "B", prob.B)
    if m:
        fails.append("input chain: " + m)
    mode = str(g["mode"])
    levels = setup.hierarchy.levels
    coarsest_n = int(g["coarsest_n"])
    if levels[-1].n != coarsest_n:
        fails.append(f"coarsest level n={levels[-1].n}, reference {coarsest_n}")
    n_kept = len(levels)
    if "n_levels" in g and n_kept != int(g["n_levels"]):
        fails.append(f"{n_kept} levels, reference {int(g['n_levels'])}")
    checked = 0
    for li, lev in enumerate(levels):
        if li >= int(g["n_entries"]):
            break
        for key, M in (("B", lev.dB), ("M", lev.dM), ("N", lev.dN)):
            msg = csr_mismatch(g, f"E{li}_{key}", M, n=lev.n)
            checked += 1
            if msg:
                fails.append(f"level {li}: {msg}")
        if lev.dP is None:
            continue
        if sha(lev.split.coarse) != str(g[f"S{li}_sha"]):
            fails.append(f"level {li}: C/F split differs")
        for key, M in (("P", lev.dP), ("Q", lev.dQ)):
            msg = csr_mismatch(g, f"{key}{li}", M)
            checked += 1
            if msg:
                fails.append(f"level {li}: {msg}")
    out = {"config": name, "mode": mode, "levels": [lv.n for lv in levels], "operators_checked": checked}
    if mode != "downward":
        fam, size, k, stop, restart, _ = bench.CONFIGS[name]
        vop = pb.VCycleOperator(setup.hierarchy, cfg.smoother)
        gcfg = pb.GmresConfig(restart=restart, rtol=bench.RTOL)
        zero = torch.zeros(prob.n, dtype=torch.float64, device="cuda")
        if mode == "full":
            start = setup.dx0
            est, low, _ = vec_errors(g, "x0", setup.dx0.cpu().numpy())
            out["x0_err_l1_est"] = est
            if est > 1e-8:
                fails.append(f"x0 l1 error ~{est:.2e}")
        else:
            start = torch.full((prob.n,), 1.0 / prob.n, dtype=torch.float64, device="cuda")
        rep = pb.gmres(dB, zero, start, gcfg, vop, to_host=False)
        its, ref_its = rep.iterations, int(g["iterations"])
        out.update(iterations=its, reference_iterations=ref_its, gmres_start=str(g["gmres_start"]))
        if abs(its - ref_its) > max(1, int(0.1 * ref_its)):
            fails.append(f"GMRES iterations {its} vs reference {ref_its}")
        x = _sign_fix_l1(rep.x_device.cpu().numpy())
        est, low, full = vec_errors(g, "x", x)
        out.update(x_err_l1=full, x_err_l1_est=est, x_err_l1_blocks=low)
        err = full if full is not None else est
        if err > 1e-8 or low > 1e-8:
            fails.append(f"x l1 error {err:.2e} (blocks {low:.2e})")
        vin = np.random.default_rng(7).standard_normal(prob.n)
        vin -= vin.mean()
        vout = vop.apply(vin)
        vout = vout.cpu().numpy() if hasattr(vout, "cpu") else np.asarray(vout)
        ref = g["vout_every64"]
        verr = float(np.abs(vout[::64] - ref).max() / max(np.abs(ref).max(), 1e-300))
        out["vcycle_err_rel"] = verr
        if verr > 1e-9:
            fails.append(f"V-cycle apply differs ({verr:.2e} relative)")
    out["failures"] = fails
    out["ok"] = not fails
    return out
