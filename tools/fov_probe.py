"""FOV diagnostics against the reference fixture, printing distances (development tool).

python tools/fov_probe.py
"""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))
from test_gpu_fov import _hausdorff, _segment_distance  # noqa: E402
from paper_1402_4005_b200.fov import eigenvalue_dots, fov_boundary  # noqa: E402

z = np.load(Path(__file__).resolve().parent.parent / "tests/golden/fov.npz")
for name in z["names"]:
    A = z[f"{name}_A"]
    t = time.time()
    f = fov_boundary(A, n_angles=int(z[f"{name}_angles"]))
    dt = time.time() - t
    lap = np.linalg.eigvals(A)
    print(f"{name:10s} n={A.shape[0]:5d} hull {f.boundary.size:3d}/{z[name + '_boundary'].size:3d} "
          f"bnd {_segment_distance(z[name + '_boundary'], f.boundary):.1e}/{_segment_distance(f.boundary, z[name + '_boundary']):.1e} "
          f"nu {abs(f.nu - float(z[name + '_nu'])):.1e} eig(ours-ref) {_hausdorff(f.eigenvalues, z[name + '_eigenvalues']):.1e} "
          f"eig(lapack-ref) {_hausdorff(lap, z[name + '_eigenvalues']):.1e} t={dt:.3f}s ref={float(z[name + '_seconds']):.3f}s",
          flush=True)
