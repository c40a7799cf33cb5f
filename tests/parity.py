"""Parity metrics (BASELINE.md §3 / SURVEY §8(d)) used by the GPU tests and
tools/parity_full.py. Pure numpy, test infrastructure only."""
from __future__ import annotations

import numpy as np

# BASELINE.json north_star tolerances
REL_ERR_ABS_TOL = 1e-10       # |rel_err_gpu - rel_err_ref|
ANGLE_TOL = 1e-8              # largest principal angle between factor subspaces
CORE_SV_REL_TOL = 1e-9        # core mode-n singular values, relative
ORTHO_TOL_PER_RANK = 1e-12    # ||U^T U - I||_F / R  (acceptance C7)


def principal_sine(u_gpu: np.ndarray, u_ref: np.ndarray) -> float:
    """sin of the largest principal angle, from the projection residual
    sigma_max(U_gpu - U_ref (U_ref^T U_gpu)); not acos of the overlap, whose
    resolution bottoms out near sqrt(eps) (test_als.cpp:59-61)."""
    resid = u_gpu - u_ref @ (u_ref.T @ u_gpu)
    if resid.size == 0:
        return 0.0
    return float(np.linalg.svd(resid, compute_uv=False)[0])


def core_mode_spectra(core: np.ndarray):
    out = []
    for n in range(core.ndim):
        unf = np.moveaxis(core, n, 0).reshape(core.shape[n], -1, order="F")
        out.append(np.linalg.svd(unf, compute_uv=False))
    return out


def core_sv_rel_diff(core_a: np.ndarray, core_b: np.ndarray) -> float:
    worst = 0.0
    for sa, sb in zip(core_mode_spectra(core_a), core_mode_spectra(core_b)):
        scale = max(float(np.max(np.abs(sb))), 1e-300)
        worst = max(worst, float(np.max(np.abs(sa - sb)) / scale))
    return worst


def ortho_defect(u: np.ndarray) -> float:
    g = u.T @ u - np.eye(u.shape[1])
    return float(np.linalg.norm(g) / u.shape[1])


def compare_decompositions(gpu_tk, gpu_rep, ref_res):
    """Returns a dict of parity metrics between the B200 result and the
    reference's (oracles.HosvdResult)."""
    angles = [principal_sine(g, r) for g, r in zip(gpu_tk.factors, ref_res.factors)]
    iters_gpu = [(m.mode, m.als.iterations) for m in gpu_rep.per_mode]
    iters_ref = [(m.mode, m.iterations) for m in ref_res.per_mode]
    return {
        "rel_err_gpu": gpu_rep.relative_residual,
        "rel_err_ref": ref_res.relative_residual,
        "rel_err_abs_diff": abs(gpu_rep.relative_residual - ref_res.relative_residual),
        "max_principal_sine": max(angles),
        "principal_sines": angles,
        "core_sv_rel_diff": core_sv_rel_diff(np.asarray(gpu_tk.core), np.asarray(ref_res.core)),
        "iters_gpu": iters_gpu,
        "iters_ref": iters_ref,
        "iters_equal": iters_gpu == iters_ref,
        "max_ortho_defect": max(ortho_defect(u) for u in gpu_tk.factors),
    }


def assert_parity(m: dict, angle_tol: float = ANGLE_TOL):
    assert m["iters_equal"], (m["iters_gpu"], m["iters_ref"])
    assert m["rel_err_abs_diff"] <= REL_ERR_ABS_TOL, m
    assert m["max_principal_sine"] <= angle_tol, m
    assert m["core_sv_rel_diff"] <= CORE_SV_REL_TOL, m
    assert m["max_ortho_defect"] <= ORTHO_TOL_PER_RANK, m


def column_diff(u_gpu: np.ndarray, u_ref: np.ndarray) -> float:
    """Largest column-wise distance between two factor matrices whose columns
    are individually determined (singular vectors under dense_svd's sign
    convention, kernels.cpp:25-43)."""
    if u_gpu.size == 0:
        return 0.0
    return float(np.max(np.linalg.norm(u_gpu - u_ref, axis=0)))


def column_alignment(w: np.ndarray, j: int, u: np.ndarray, k: int) -> float:
    """|<w_j, u_k>| / (|w_j| |u_k|) (test_hosvd.cpp column_alignment)."""
    a, b = w[:, j], u[:, k]
    return float(abs(a @ b) / (np.linalg.norm(a) * np.linalg.norm(b)))
