"""Full-size parity for configs 3 and 4 against the unmodified reference
(fixtures from tests/golden/make_golden_large.py, run in the build
container with a chunked on-the-fly operator adapter), plus size-independent
properties at full size: orthonormal bases, the BASELINE gates estimated
with fixed Gaussian probes W (E||X w||^2 = ||X||_F^2)."""

import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_2501_05528_b200 as P
from cases import GOLDEN, probe_vec

pytestmark = pytest.mark.gpu


def _fixture(name):
    path = os.path.join(GOLDEN, name + ".npz")
    if not os.path.exists(path):
        pytest.skip(f"{name} fixture not generated")
    return dict(np.load(path))


@pytest.mark.parametrize("name,mid", [("c3_A1", "A1"), ("c4_B2", "B2")])
def test_fullsize_against_reference(name, mid):
    g = _fixture(name)
    pts = P.grid_points(256, 2)
    tess = P.build_tessellation(pts, 256)
    op = P.KernelOperator(pts, "log", -np.log(0.5 / 256))
    rep, report = P.compress(op, tess, 40, mid, p=10, stream=P.RandomStream(7), compute_error=False)
    W = np.stack([probe_vec(tess.n_points, 10 + c) for c in range(3)], axis=1)
    scale = float(g["A_fro"]) * np.sqrt(W.shape[1])
    AW = rep.apply(W)
    AtW = rep.apply_adjoint(W)
    # ||A_hat_gpu - A_hat_ref||_F / ||A||_F  (probe estimate)
    tol = 1e-10
    if mid == "B2":
        # B2 at this size is rounding-sensitive: moving every grid coordinate
        # by one ulp (A entries change by ~1e-16 relative) moves OUR OWN A_hat
        # by ~4.6e-9 (measured on B200, tools/diag_b2_sens.py), the same order
        # as the distance to the reference. No implementation that does not
        # reproduce numpy's floating-point operations bit for bit can meet
        # 1e-10 here; the gate becomes 3x the measured rounding sensitivity
        # and the 1.05x approximation-error gate below stays.
        op2 = P.KernelOperator(np.nextafter(pts.coords, 2.0), "log", -np.log(0.5 / 256))
        rep2, _ = P.compress(op2, tess, 40, mid, p=10, stream=P.RandomStream(7), compute_error=False)
        sens = np.linalg.norm(AW - rep2.apply(W)) / scale
        tol = max(tol, 3.0 * sens)
    assert np.linalg.norm(AW - g["Ahat_W"]) / scale <= tol
    assert np.linalg.norm(AtW - g["Ahat_tW"]) / scale <= tol
    # approximation error within 1.05x of the reference's
    err_gpu = np.linalg.norm(g["A_W"] - AW)
    err_ref = np.linalg.norm(g["A_W"] - g["Ahat_W"])
    assert err_gpu <= 1.05 * err_ref + 1e-12 * scale
    mv = np.array([[report.matvecs.get(ph, {"A": 0})["A"], report.matvecs.get(ph, {"Astar": 0})["Astar"]]
                   for ph in ("I", "II", "III")])
    assert np.array_equal(mv, g["matvecs"])


def test_fullsize_c5_shard_properties():
    """One 1/8 row shard of config 5: orthonormal U, finite core, near blocks
    consistent with the emulated single-process pipeline on the same shard."""
    from paper_2501_05528_b200.distributed import phase1_local, shard_ranges
    pts = P.grid_points(1024, 2)
    tess = P.build_tessellation(pts, 4096)
    op = P.KernelOperator(pts, "inv", 2048.0)
    sh = shard_ranges(tess, 8, 48)[3]
    plan = P.plan_tagging(tess, 0, "gaussian", P.RandomStream(7).child(1))
    _, U, V, dt = phase1_local(op, tess, 48, 16, P.RandomStream(7), sh, plan)
    m = 256
    Ub = U.reshape(-1, m, 48)
    G = torch.bmm(Ub.transpose(1, 2), Ub)
    eye = torch.eye(48, dtype=torch.float64, device=G.device)
    assert float((G - eye).abs().max()) <= 1e-12
    Vb = V.reshape(-1, m, 48)
    assert float((torch.bmm(Vb.transpose(1, 2), Vb) - eye).abs().max()) <= 1e-12
