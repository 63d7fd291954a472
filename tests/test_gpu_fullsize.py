"""Full-size parity for configs 3 and 4 against the unmodified reference
(fixtures from tests/golden/make_golden_large.py, run in the build container
with a chunked on-the-fly operator adapter).

Gates (BASELINE.json north star):
* ||A - A_hat_gpu||_F <= 1.05 ||A - A_hat_ref||_F, both EXACT: the GPU side by
  ublr_frob_error (every block pair, A generated on the device), the
  reference side computed blockwise in the build container and stored;
* ||A_hat_gpu - A_hat_ref||_F / ||A||_F <= 1e-10 (c3). The reference's 2 GB
  output cannot travel to the GPU box, so this distance is estimated from 8
  fixed Gaussian probe columns W in both directions (E||X W||_F^2 =
  8 ||X||_F^2), with the estimator's own spread added (upper 3-sigma bound
  over the 16 column estimates).
* c4 (B2) is rounding-sensitive IN THE REFERENCE ITSELF: moving every grid
  coordinate by one ulp (A entries change by ~1e-16 relative) moves the
  unmodified reference's A_hat by ||A_hat_ref - A_hat_ref'||_F / ||A||_F =
  7.9e-9 (exact, `sens_fro` in the fixture), 79x the 1e-10 gate and above the
  reference's own approximation error (7.5e-9). Two implementations that
  round differently are two such perturbations, so the c4 parity gate is
  2 x the reference's own sensitivity — a fixed number from the reference,
  not from this implementation. What the reference's B2
  error consists of: 95 % of its ||A - A_hat||_F^2 sits in the far field, 87 %
  in three block rows of the core (fixture `err_pair`), the rows of the near
  pairs whose projected tag (the type-B denominator) is 4e-4 .. 1.2e-3
  against a median of 0.66 -- the sketch's rounding noise
  divided by that denominator and pushed through the core least squares. It
  is a rounding-noise level, not a truncation error, so a single run is one
  draw (two runs of the unmodified reference that differ only in the BLAS
  threading of the operator adapter give 7.49e-9 and 7.11e-9). The GPU path
  removes the largest noise term (compensated fold of the tagged sketch,
  compensated pair combination) and must meet BOTH forms of the 1.05x gate:
  the unperturbed run against the reference's unperturbed run, and the
  root-mean-square exact error over the same family of five 1-ulp
  coordinate perturbations on both sides (fixture `err_family`).
The c5 spot checks are in test_gpu_c5_parity.py."""

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
    g = dict(np.load(path))
    if "err_fro" not in g:
        pytest.skip(f"{name} fixture predates the exact-norm format")
    return g


def probe_distance_bound(rep, g):
    """Upper 3-sigma bound of ||A_hat_gpu - A_hat_ref||_F from the probe columns."""
    ncol = g["Ahat_W"].shape[1]
    W = np.stack([probe_vec(rep.n, 10 + c) for c in range(ncol)], axis=1)
    d1 = rep.apply(W) - g["Ahat_W"]
    d2 = rep.apply_adjoint(W) - g["Ahat_tW"]
    per_col = np.concatenate([np.sum(d1 * d1, axis=0), np.sum(d2 * d2, axis=0)])   # each estimates ||dA||_F^2
    mean = per_col.mean()
    sem = per_col.std(ddof=1) / np.sqrt(per_col.size)
    return np.sqrt(mean + 3.0 * sem), np.sqrt(mean)


@pytest.mark.parametrize("name,mid", [("c3_A1", "A1"), ("c4_B2", "B2")])
def test_fullsize_against_reference(name, mid):
    g = _fixture(name)
    pts = P.grid_points(256, 2)
    tess = P.build_tessellation(pts, 256)
    op = P.KernelOperator(pts, "log", -np.log(0.5 / 256))
    rep, report = P.compress(op, tess, 40, mid, p=10, stream=P.RandomStream(7), compute_error=False)
    A_fro = float(g["A_fro"])
    # approximation error: exact on both sides
    fr = P.frobenius_error(op, rep)
    assert fr.ref_fro == pytest.approx(A_fro, rel=1e-12)
    err_gpu, err_ref = fr.fro / A_fro, float(g["err_fro"]) / A_fro
    print(f"{name}: ||A - A_hat||_F / ||A||_F gpu {err_gpu:.4e} ref {err_ref:.4e} ({err_gpu / err_ref:.3f}x)")
    assert err_gpu <= 1.05 * err_ref
    if mid == "B2":
        # rms of the exact error over the same family of 1-ulp coordinate
        # perturbations on both sides (each against the unperturbed A)
        assert "err_family" in g, "c4 fixture lacks the reference's perturbation family"
        names = [str(x) for x in g["err_family_names"]]
        c = pts.coords
        variants = {"base": c, "+1ulp": np.nextafter(c, 2.0), "-1ulp": np.nextafter(c, -1.0),
                    "+1ulp x": np.stack([np.nextafter(c[:, 0], 2.0), c[:, 1]], 1),
                    "+2ulp": np.nextafter(np.nextafter(c, 2.0), 2.0)}
        errs = []
        for nm in names:
            if nm == "base":
                errs.append(err_gpu)
                continue
            rv, _ = P.compress(P.KernelOperator(variants[nm], "log", -np.log(0.5 / 256)), tess, 40, mid, p=10,
                               stream=P.RandomStream(7), compute_error=False)
            errs.append(P.frobenius_error(op, rv).fro / A_fro)
            rv = None
        ref_errs = np.asarray(g["err_family"], dtype=float) / A_fro
        rms_gpu, rms_ref = np.sqrt(np.mean(np.square(errs))), np.sqrt(np.mean(np.square(ref_errs)))
        print(f"{name}: exact errors over {names}: gpu {np.round(np.array(errs) * 1e9, 3)} e-9, "
              f"ref {np.round(ref_errs * 1e9, 3)} e-9; rms gpu {rms_gpu:.4e} ref {rms_ref:.4e} "
              f"({rms_gpu / rms_ref:.3f}x)")
        assert rms_gpu <= 1.05 * rms_ref
    # parity distance to the reference (probe estimate, upper bound)
    bound, est = probe_distance_bound(rep, g)
    tol = 1e-10 if mid != "B2" else 2.0 * float(g["sens_fro"]) / A_fro
    print(f"{name}: ||A_hat_gpu - A_hat_ref||_F / ||A||_F ~ {est / A_fro:.3e} (3-sigma bound {bound / A_fro:.3e}, "
          f"gate {tol:.2e})")
    assert bound / A_fro <= tol
    mv = np.array([[report.matvecs.get(ph, {"A": 0})["A"], report.matvecs.get(ph, {"Astar": 0})["Astar"]]
                   for ph in ("I", "II", "III")])
    assert np.array_equal(mv, g["matvecs"])
    assert report.storage_entries == int(g["storage_entries"])


def test_fullsize_c4_own_sensitivity_below_reference():
    """The GPU B2 path's own 1-ulp sensitivity (exact, ublr_frob_diff) is of
    the reference's size (within 1.5x of the fixture's `sens_fro`, same
    perturbation): the GPU arithmetic does not amplify rounding more."""
    g = _fixture("c4_B2")
    pts = P.grid_points(256, 2)
    tess = P.build_tessellation(pts, 256)
    diag = -np.log(0.5 / 256)
    rep, _ = P.compress(P.KernelOperator(pts, "log", diag), tess, 40, "B2", p=10, stream=P.RandomStream(7),
                        compute_error=False)
    rep2, _ = P.compress(P.KernelOperator(np.nextafter(pts.coords, 2.0), "log", diag), tess, 40, "B2", p=10,
                         stream=P.RandomStream(7), compute_error=False)
    sens = P.frobenius_distance(rep, rep2).fro
    print(f"c4 B2 1-ulp sensitivity / ||A||_F: gpu {sens / float(g['A_fro']):.3e} "
          f"ref {float(g['sens_fro']) / float(g['A_fro']):.3e}")
    assert sens <= 1.5 * float(g["sens_fro"])
